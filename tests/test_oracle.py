"""Pin the C oracle (oracle/lsv_oracle.c) against an independent float64 restatement.

The reference has no LoRA arithmetic, so the delta oracle's parity is UNPINNED by
the reference; these tests pin the oracle to the math itself."""

import numpy as np
import pytest

from oracle import oracle
from tests._cases import Case


@pytest.mark.parametrize("lengths,ranks", [
    ([64, 64, 64, 64], [8, 16, 64, 128]),          # config 1 shape
    ([1, 0, 5, 17], [8, 32, 24, 128]),             # ragged + empty segment
])
def test_c_oracle_matches_float64(lengths, ranks):
    case = Case(512, 384, lengths, ranks, seed=11)
    c = case.oracle_delta()
    f = case.oracle_delta_f64()
    assert oracle.max_rel_err(c, f) < 1e-5
    n = case.seg.num_tokens
    assert np.all(c[n:] == 0)


def test_c_oracle_threads_independent():
    case = Case(256, 256, [9, 30, 2], [8, 16, 64], seed=12)
    a = oracle.delta_c(*_args(case), threads=1)
    b = oracle.delta_c(*_args(case), threads=4)
    assert np.array_equal(a, b)


def test_bf16_roundtrip_helpers():
    x = np.array([1.0, -2.5, 3.1415926, 1e-3, 65504.0], dtype=np.float32)
    bits = oracle.f32_to_bf16_bits(x)
    back = oracle.bf16_bits_to_f32(bits)
    assert np.allclose(back, x, rtol=2 ** -8)
    assert np.array_equal(oracle.f32_to_bf16_bits(back), bits)


def test_max_rel_err_metric():
    ref = np.array([[1.0, -4.0], [0.0, 2.0]])
    assert oracle.max_rel_err(ref, ref) == 0.0
    assert oracle.max_rel_err(ref + 0.04, ref) == pytest.approx(0.01)


def _args(case):
    from tests._cases import bf16_bits
    return (bf16_bits(case.x), case.seg.seg_indptr, case.seg.seg_rank,
            [bf16_bits(a) for a in case.a], [bf16_bits(b) for b in case.b], case.h_out)
