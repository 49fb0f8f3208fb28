"""The GPU parity subset on the bounds-checked library build.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs
needing a reset), so memory-safety evidence comes from libevsim_gpu_checked.so:
the same sources compiled with -DEVSIM_CHECKED, where every chain kernel's
mask / count stores, the emit's tile and staging bounds and the LK solver's
patch-grid stores are checked on the device (evsim_device.cuh EVSIM_CHECK;
a violation prints the site and traps).  The checked library runs the
golden-fixture parity tests (every method, both contrast modes, magnitude,
no endpoints), the pipelined / long pushes, the stacked streams and the
tile-staged chain in a subprocess (EVSIM_GPU_LIB=checked) and must pass bit-exact with no trap.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2209_04634_b200", "libevsim_gpu_checked.so")


def test_checked_library_exports_the_abi():
    """CPU: the checked build exists and exports the same C-ABI."""
    if not os.path.exists(CHECKED):
        pytest.skip("checked build missing (build.py checked=True)")
    out = subprocess.run(["nm", "-D", "--defined-only", CHECKED], capture_output=True, text=True).stdout
    from paper_2209_04634_b200 import _lib
    for name in _lib.EXPORTED:
        assert f" {name}" in out, name


@pytest.mark.gpu
def test_parity_subset_on_checked_build():
    if not os.path.exists(CHECKED):
        pytest.skip("checked build missing")
    env = dict(os.environ, EVSIM_GPU_LIB="checked")
    sel = ("test_gpu_matches_reference_golden or test_pipelined_dense_push_matches_oracle or "
           "test_stacked_streams_equal_per_stream_oracle or test_streaming_difference_chain_long_push or "
           "test_sequence_pipelined_push_matches_reference or test_tile_chain_matches_oracle or "
           "test_tile_chain_noise_flow or test_tile_chain_sizes")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider", "-k", sel,
                        "tests/test_gpu_parity.py", "tests/test_gpu_batch.py", "tests/test_gpu_stacked.py",
                        "tests/test_gpu_sequences.py", "tests/test_gpu_tile_chain.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout[-4000:] + r.stderr[-4000:])
    assert r.returncode == 0, tail
    assert "EVSIM_CHECKED" not in r.stdout + r.stderr, tail
    assert " passed" in r.stdout, tail
