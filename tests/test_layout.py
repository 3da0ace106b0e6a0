"""The chain-interleaved row layout of the reference-order distances
(csrc/pag_device.h chain_positions / chain_xstride, pag_util.cu
interleave_rows_kernel, pag_search.cu dist_exact_x), restated in numpy and
checked on the CPU against the oracle's sq_dist (vecstore.cpp:77-95) bit for
bit: running each chain serially over its 8-float runs of every 128-B line,
tail elements as extra chain-0 positions, zero padding, gives the reference
sum for any padded_dim. The GPU parity tests check the kernels themselves."""
import numpy as np
import pytest

from oracle import oracle as O


def chain_xstride(padded: int) -> int:
    positions = padded // 4 + padded % 4
    return (positions + 7) // 8 * 32


def interleave(row: np.ndarray) -> np.ndarray:
    padded = row.shape[0]
    d4 = padded & ~3
    out = np.zeros(chain_xstride(padded), dtype=np.float32)
    for k in range(padded):
        p, c = (k // 4, k % 4) if k < d4 else (d4 // 4 + (k - d4), 0)
        out[(p // 8) * 32 + 8 * c + p % 8] = row[k]
    return out


def chain_sq_dist(xrow: np.ndarray, xq: np.ndarray) -> np.float32:
    acc = [np.float32(0)] * 4
    for line in range(xrow.shape[0] // 32):
        for c in range(4):
            for i in range(8):
                j = 32 * line + 8 * c + i
                d = np.float32(xrow[j] - xq[j])
                acc[c] = np.float32(acc[c] + np.float32(d * d))
    return np.float32(np.float32(acc[0] + acc[1]) + np.float32(acc[2] + acc[3]))


@pytest.mark.parametrize("dim", [1, 2, 3, 4, 5, 7, 9, 10, 30, 31, 32, 33, 48, 63, 100, 128, 131])
def test_chain_layout_reproduces_reference_order(dim):
    rng = np.random.default_rng(dim)
    base = rng.standard_normal((6, dim)).astype(np.float32)
    q = rng.standard_normal((1, dim)).astype(np.float32)
    ids, sq = O.ground_truth(base, q, 6)  # reference-order sq_dist of every row
    want = np.empty(6, dtype=np.float32)
    want[ids[0]] = sq[0]
    xq = interleave(q[0])
    got = np.array([chain_sq_dist(interleave(r), xq) for r in base], dtype=np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_xstride_is_whole_lines_and_covers_every_position():
    for padded in range(1, 200):
        xs = chain_xstride(padded)
        assert xs % 32 == 0 and xs // 4 >= padded // 4 + padded % 4 and xs >= padded
