"""The in-process multi-device C++ driver (include/oiobf/sharded.hpp): one
library handle per rank, the exchange as peer copies, host code in C++ only.
On a one-GPU box every rank sits on device 0 (the ranks run one after the
other, so none waits on another); G must equal the single-GPU contraction of
the same operator."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2411_03029_b200")
EXE = os.path.join(PKG, "_build", "sharded_test")


def _build():
    from paper_2411_03029_b200.build import build
    build()
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O1", "-pthread", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "include", "eigen_shim"), os.path.join(ROOT, "tests", "cpp", "sharded_test.cpp"),
           "-L" + PKG, "-ltbf_b200", "-Wl,-rpath," + PKG, "-o", EXE]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_sharded_headers_compile():
    _build()
    assert subprocess.run([EXE, "--compile-only"]).returncode == 0


def test_balanced_owners_cpp_equals_python():
    """The C++ driver's balanced_owners (sharded.hpp) and the Python one
    (sharded.py) compute the same ownership map -- ranks in one job may mix the
    two orchestrations only if they agree."""
    import numpy as np

    from paper_2411_03029_b200.sharded import balanced_owners
    _build()
    rng = np.random.default_rng(5)
    for n, world in ((64, 8), (64, 4), (8, 2), (16, 3), (8, 8), (12, 5)):
        w = rng.integers(10, 90, n).astype(np.float64)
        w[: n // 4] *= 3
        w[n // 2] = w[n // 2 + 1]  # a tie
        r = subprocess.run([EXE, "--owners", str(world)] + [repr(float(x)) for x in w], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-500:]
        assert json.loads(r.stdout.strip()) == balanced_owners(w, world).tolist(), (n, world)


@pytest.mark.gpu
@pytest.mark.parametrize("world,case", [(2, "cubes32"), (4, "cubes32"), (8, "cubes32"), (3, "radon64"),
                                        (8, "plates64L4"), (4, "dft6")])
def test_sharded_cpp_matches_single_gpu(world, case):
    _build()
    r = subprocess.run([EXE, str(world), case], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["world"] == world
    assert out["rel"] < 1e-12, out


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_cpp_balanced_ownership(world):
    """tbf_construct_sharded_balanced: the LPT ownership map of the measured
    per-s core bytes gives the same G and a heaviest rank no heavier than
    round-robin's."""
    _build()
    outs = []
    for mode in ("", "balanced"):
        r = subprocess.run([EXE, str(world), "cubes32"] + ([mode] if mode else []), capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    rr, bal = outs
    assert rr["rel"] < 1e-12 and bal["rel"] < 1e-12, outs
    assert bal["core_max_over_mean"] <= rr["core_max_over_mean"] + 1e-12, outs
