"""BenchRecord CSV: fixed header, fieldwise-exact round
trip (CPU), and the spec's run_single examples on the GPU."""
import numpy as np
import pytest

from paper_2411_03029_b200.records import HEADER, BenchRecord, emit_csv, parse_csv


def _rec(i, err=1.25e-7):
    return BenchRecord("green", 2, 64, 1e-6, "tensor-bf", 2, 0.0123 + i, 4.5e-5, 123456789, 10, 4, err, 3, 1)


def test_csv_header_fixed():
    assert HEADER == ["kernel", "d", "n", "tol", "algo", "L", "factor_time_s", "apply_time_s", "memory_bytes", "r",
                      "r_min", "rel_error", "seed", "n_v"]


def test_csv_empty_and_single(tmp_path):
    p = tmp_path / "e.csv"
    emit_csv([], p)
    assert p.read_text().splitlines() == [",".join(HEADER)]
    assert parse_csv(p) == []
    emit_csv([_rec(0)], p)
    assert len(p.read_text().splitlines()) == 2


def test_csv_roundtrip_fieldwise_exact(tmp_path):
    rng = np.random.default_rng(0)
    recs = [_rec(i, err=float(rng.random()) * 1e-3) for i in range(5)] + [_rec(9, err=None)]
    p = tmp_path / "r.csv"
    emit_csv(recs, p)
    assert parse_csv(p) == recs


@pytest.mark.gpu
def test_run_single_spec_examples():
    from paper_2411_03029_b200.configs import dft, green_plates
    from paper_2411_03029_b200.records import run_single
    r = run_single(dft(1, 64, bitrev=False), 1e-6, 2)
    assert r.rel_error <= 1e-4 and r.algo == "tensor-bf" and r.memory_bytes > 0
    ranks = [run_single(green_plates(64), tol, 2).r for tol in (1e-2, 1e-3, 1e-4, 1e-5)]
    assert all(a <= b for a, b in zip(ranks, ranks[1:])), ranks
    assert run_single(green_plates(16), 1e-6, 2, algo="dense").rel_error <= 1e-13
