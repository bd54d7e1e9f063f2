"""The -DMMF_DEBUG build (libmmf_debug.so: device-side checks of ring slots, CSR / ELL indices and message exponents,
csrc/xf.cuh MMF_DASSERT) over a representative slice of the GPU parity suite — the memory-safety net in place of
compute-sanitizer, which this pool does not offer.  A failed check traps the kernel (MMF_ECUDA)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUBSET = ("micro_parity or tiny_config1 or ragged or pipelined_kernels_L1024 or hub_and_empty or "
          "pipelined_time_varying or large_ratio or node_caps_parity or commodity_times_parity or symmetric_gs_parity "
          "or node_costs_parity or virtual_ranks or wide_lane_multi_group")


def test_debug_build_runs_the_parity_subset_clean():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2106_14485_b200.build import build
    lib = build(debug=True)
    env = dict(os.environ, MMF_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", SUBSET],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert "MMF_DEBUG check failed" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    assert " passed" in out
