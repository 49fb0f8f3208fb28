"""The C++ drop-in header include/evsim_b200.hpp: compiles against the C-ABI,
host-side semantics on CPU, and (GPU) push_frame / push_frames parity with the
oracle through C++."""
import os
import subprocess

import numpy as np
import pytest

from helpers import assert_same_events, concat, run_oracle_stream
from paper_2209_04634_b200 import _lib
from paper_2209_04634_b200.abi import EVENT_DTYPE, Method, make_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "wrapper_check.cpp")
LIBDIR = os.path.dirname(_lib.LIB_PATH)


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    _lib.load()  # builds the library if needed
    out = str(tmp_path_factory.mktemp("cpp") / "wrapper_check")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include", SRC, "-o", out,
                    f"-L{LIBDIR}", "-levsim_gpu", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return out


def test_cpp_header_compiles_and_host_semantics(binary):
    r = subprocess.run([binary, "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "cpu checks ok" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("method,mode", [(Method.dense, 1), (Method.sparse, 0), (Method.difference_only, 1),
                                         (Method.difference_interp, 0)])
def test_cpp_push_parity(binary, oracle, tmp_path, method, mode):
    from paper_2209_04634_b200 import scenes
    frames, ts = scenes.generate("c2", n_frames=5, width=120, height=90)
    n, h, w = frames.shape
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        f.write(np.array([w, h, n, int(method), mode], np.int32).tobytes())
        f.write(frames.tobytes())
        f.write(ts.astype(np.int64).tobytes())
    o1, o2 = tmp_path / "o1.bin", tmp_path / "o2.bin"
    r = subprocess.run([binary, "gpu", str(inp), str(o1), str(o2)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    cfg = make_config(method, contrast_mode=mode)
    exp = concat(run_oracle_stream(oracle, cfg, frames, ts))
    for o in (o1, o2):
        got = np.frombuffer(open(o, "rb").read(), dtype=EVENT_DTYPE)
        assert_same_events(got, exp)
