"""Kernel catalog — CPU checks of the
oracle's entry functors against independent numpy restatements of the paper
formulas, plus the spec's catalog invariants (unit modulus of phase kernels,
determinism, NUDFT locations in [0, n-1]).  The device functors are checked
against the oracle entrywise in tests/test_gpu_parity.py."""
import numpy as np
import pytest

from paper_2411_03029_b200.configs import dft, green_cubes, green_plates, nudft, radon2d, radon3d


def _pairs(spec, count, seed):
    rng = np.random.default_rng(seed)
    I = rng.integers(1, spec.n + 1, size=(count, spec.d))
    J = rng.integers(1, spec.n + 1, size=(count, spec.d))
    return I.astype(np.int64), J.astype(np.int64)


def test_radon3d_formula(oracle):
    spec = radon3d(32)
    I, J = _pairs(spec, 500, 1)
    got = oracle.kernel_eval(spec, I, J)
    n = spec.n
    x = (I - 1) / n
    k = (J - 1 - n // 2).astype(np.float64)
    c = (3 + np.prod(np.sin(2 * np.pi * x), axis=1)) / 100
    frac = np.mod(np.sum((I - 1) * (J - 1 - n // 2), axis=1), n) / n  # x.k reduced exactly mod 1
    phi = frac + c * np.sqrt(np.sum(k * k, axis=1))
    np.testing.assert_allclose(got, np.exp(2j * np.pi * phi), rtol=0, atol=1e-12)
    # x = 0 (i = 1): c = 3/100 exactly
    e = oracle.kernel_eval(spec, np.array([[1, 1, 1]]), np.array([[n // 2 + 4, n // 2 + 1, n // 2 + 1]]))
    np.testing.assert_allclose(e, np.exp(2j * np.pi * 0.03 * 3), atol=1e-14)


def test_nudft_formula_and_locations(oracle):
    spec = nudft(2, 32, seed=7)
    I, J = _pairs(spec, 500, 2)
    got = oracle.kernel_eval(spec, I, J)
    n = spec.n
    flat = (I[:, 0] - 1) + n * (I[:, 1] - 1)
    x = np.zeros((len(I), 2))
    for e in range(len(I)):
        for k in range(2):
            h = oracle.derive_seed(7, [0x4E, int(flat[e]), k])
            x[e, k] = float(h >> 11) * 2.0 ** -53 * (n - 1)
    assert np.all((x >= 0) & (x <= n - 1))
    phi = np.sum(x * (J - 1) / n, axis=1)
    np.testing.assert_allclose(got, np.exp(2j * np.pi * phi), rtol=0, atol=1e-10)
    # a different seed moves the locations
    other = oracle.kernel_eval(nudft(2, 32, seed=8), I, J)
    assert np.max(np.abs(other - got)) > 0.1


@pytest.mark.parametrize("spec", [radon2d(16), radon3d(8), dft(3, 8), dft(1, 16), nudft(2, 16, 3)],
                         ids=["radon2d", "radon3d", "dft3", "dft1", "nudft2"])
def test_phase_kernels_unit_modulus_and_deterministic(oracle, spec):
    I, J = _pairs(spec, 1000, 3)
    a = oracle.kernel_eval(spec, I, J)
    b = oracle.kernel_eval(spec, I, J)
    assert np.array_equal(a, b)
    assert np.max(np.abs(np.abs(a) - 1)) <= 1e-14


def test_green_translational_invariance(oracle):
    spec = green_plates(32)
    I, J = _pairs(spec, 200, 4)
    shift = np.array([3, -2])
    ok = np.all((I + shift >= 1) & (I + shift <= 32) & (J + shift >= 1) & (J + shift <= 32), axis=1)
    a = oracle.kernel_eval(spec, I[ok], J[ok])
    b = oracle.kernel_eval(spec, I[ok] + shift, J[ok] + shift)
    np.testing.assert_allclose(a, b, rtol=1e-12)
    assert green_cubes(8).d == 3


def test_dft_d1_is_the_dft_matrix(oracle):
    """SPEC.md:364 example: DFT d = 1 without reordering is the DFT matrix
    (in this catalog's sign/origin convention, App. A1)."""
    n = 8
    spec = dft(1, n, bitrev=False)
    I, J = np.meshgrid(np.arange(1, n + 1), np.arange(1, n + 1), indexing="ij")
    got = oracle.kernel_eval(spec, I.reshape(-1, 1), J.reshape(-1, 1)).reshape(n, n)
    ref = np.exp(-2j * np.pi * (I - 1) * (J - 1 - n // 2) / n)
    np.testing.assert_allclose(got, ref, atol=1e-14)
