"""CPU: the C-ABI library loads and exports exactly what include/evsim_gpu.h declares.

No compute calls (no GPU here); only the pure-host entry points
(config defaults / validation) are exercised.
"""
import ctypes
import os
import re

import pytest

from paper_2209_04634_b200 import _lib
from paper_2209_04634_b200.abi import CConfig, Method, defaults

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "evsim_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"EVSIM_GPU_API\s+[\w\s\*]+?\b(evsim_gpu_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "evsim_gpu_push_frame" in names and "evsim_gpu_dense_flow" in names
    assert len(names) == 41


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(_lib.EXPORTED)


def test_library_exports_nothing_else():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted(l.split()[-1] for l in out.splitlines() if " T " in l and "evsim" in l)
    assert exported == declared_functions()


@pytest.mark.parametrize("m", list(Method))
def test_config_defaults_match_reference(m):
    # SimulatorConfig::defaults, reference include/evsim/types.hpp:101-120
    c = CConfig()
    _lib.load().evsim_gpu_config_defaults(int(m), ctypes.byref(c))
    d = defaults(m)
    for k in ("method", "c_pos", "c_neg", "n_interp", "flow_preset", "selection_threshold",
              "events_per_crossing", "include_endpoints", "contrast_mode"):
        assert getattr(c, k) == d[k], k
    table = {Method.difference_only: (2, -2, 0), Method.dense: (2, -2, 10), Method.sparse: (10, -10, 10),
             Method.difference_interp: (20, -20, 10)}
    assert (c.c_pos, c.c_neg, c.n_interp) == table[m]


@pytest.mark.parametrize("field,value,msg", [
    ("c_pos", 0, "SimulatorConfig: c_pos must be > 0"),
    ("c_neg", 0, "SimulatorConfig: c_neg must be < 0"),
    ("n_interp", -1, "SimulatorConfig: n_interp must be >= 0"),
])
def test_config_validate_messages(field, value, msg):
    from paper_2209_04634_b200 import InvalidArgument, SimulatorConfig
    cfg = SimulatorConfig.defaults(Method.dense)
    setattr(cfg, field, value)
    with pytest.raises(InvalidArgument) as e:
        cfg.validate()
    assert str(e.value) == msg


def test_log_mode_threshold_validation():
    from paper_2209_04634_b200 import ContrastMode, InvalidArgument, SimulatorConfig
    cfg = SimulatorConfig.defaults(Method.dense)
    cfg.contrast_mode = ContrastMode.log
    cfg.c_neg_log = 0.1
    with pytest.raises(InvalidArgument, match="c_neg_log must be < 0"):
        cfg.validate()


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product path fails loudly (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2209_04634_b200 import EvsimError, Simulator, SimulatorConfig
    with pytest.raises(EvsimError) as e:
        Simulator(SimulatorConfig.defaults(Method.dense))
    assert e.value.code == 3
