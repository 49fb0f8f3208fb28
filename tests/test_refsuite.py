"""The reference's OWN unit suites run against the drop-in.

/root/reference/proj/tests/test_core.cpp, test_flow.cpp and test_simulate.cpp
are compiled UNCHANGED (oracle/Makefile `refsuite`, built by
__graft_entry__.build() where /root/reference exists) against
tests/refsuite/include/evsim/*.hpp — headers that resolve every evsim:: name
to include/evsim_b200.hpp, i.e. to libevsim_gpu.so — with the
doctest-compatible harness tests/refsuite/doctest/doctest.h.  The binaries
(oracle/_ref/refsuite/, git-ignored) travel to the GPU box with the snapshot;
/root/reference is not read at run time.

Reference suites: test_core.cpp:29-200 (difference_frame, threshold_events,
config defaults), test_flow.cpp:25-207 (dense / sparse flow), and
test_simulate.cpp:30-355 (Simulator::push_frame for every method,
interpolate_frames, simulate_dense / simulate_sparse / simulate_difference,
the flow-estimator plug-in seam).
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "refsuite")
SUITES = ["test_core", "test_flow", "test_simulate"]
SUMMARY = re.compile(r"\[refsuite\] test cases: (\d+) \| passed: (\d+) \| failed: (\d+) ; "
                     r"assertions: (\d+) \| failed: (\d+)")


def _binary(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time: make -C oracle refsuite)")
    return path


def test_refsuite_binaries_link_the_b200_library():
    """CPU: every built suite binary resolves its evsim calls to libevsim_gpu.so."""
    built = [s for s in SUITES if os.path.exists(os.path.join(BIN, s))]
    if not built:
        pytest.skip("reference suites not built")
    for s in built:
        out = subprocess.run(["ldd", os.path.join(BIN, s)], capture_output=True, text=True).stdout
        assert "libevsim_gpu.so" in out, out
        assert os.path.join("paper_2209_04634_b200", "libevsim_gpu.so") in out or "not found" not in out, out


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_the_drop_in(suite):
    r = subprocess.run([_binary(suite)], capture_output=True, text=True, timeout=900, cwd=ROOT)
    m = SUMMARY.search(r.stdout)
    assert m, f"no summary line\nstdout:\n{r.stdout[-3000:]}\nstderr:\n{r.stderr[-3000:]}"
    cases, passed, failed, asserts, afailed = map(int, m.groups())
    print(m.group(0))
    assert cases > 0 and asserts > 0
    assert failed == 0 and afailed == 0 and r.returncode == 0, r.stderr[-6000:]


@pytest.mark.gpu
def test_gpu_flow_plugs_into_the_reference_simulator():
    """INTEGRATION.md §4 compiled: GpuPatchFlow / GpuLucasKanade (C-ABI flow)
    inside the reference's own Simulator (oracle/_ref) give the events of its
    default CPU estimators (dense lq / hq, sparse, magnitude without
    endpoints; tests/cpp/flow_plugin_check.cpp)."""
    path = os.path.join(ROOT, "oracle", "_ref", "flow_plugin_check")
    if not os.path.exists(path):
        pytest.skip("flow_plugin_check not built (make -C oracle plugin)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout)
    assert r.returncode == 0 and "[plugin] ok" in r.stdout, r.stdout + r.stderr
