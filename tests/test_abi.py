"""C-ABI library checks that need no GPU: the .so builds/loads and exports every declared symbol."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mmf.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mmf_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2106_14485_b200.build import build
    build()
    from paper_2106_14485_b200 import _lib
    return _lib.load()


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ["mmf_create", "mmf_set_graph", "mmf_set_costs", "mmf_set_capacity", "mmf_set_marginals",
              "mmf_set_point_marginals", "mmf_init", "mmf_sweep", "mmf_sync", "mmf_read_edge_flows",
              "mmf_read_cap_duals", "mmf_read_stats", "mmf_destroy", "mmf_last_error", "mmf_attach_nccl"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2106_14485_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mmf_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    assert set(_lib.EXPORTS) == set(declared_functions())


def test_library_is_sm100a(lib):
    from paper_2106_14485_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_null_safety(lib):
    from paper_2106_14485_b200 import _lib
    assert "mmf" in _lib.mmf_version()
    assert lib.mmf_destroy(None) == 0          # safe on NULL
    assert lib.mmf_init(None) == 2             # MMF_EINVAL


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2106_14485_b200 import _lib
    with pytest.raises(_lib.MMFError) as e:
        _lib.mmf_create(0, _lib.MMF_FP32, 0)
    assert e.value.name == "MMF_ECUDA"
