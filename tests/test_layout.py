"""K9 packing (layout.py): the vectorised path equals the per-item checked
path, and malformed input raises the reference's DataValidationError
(tuner.py:36-52 / features.py:70-92 shapes)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import Seq, random_seqs
from paper_2304_05430_b200.errors import DataValidationError
from paper_2304_05430_b200.layout import _native, _pack_checked, _pack_fast, _pack_native, pack_sequences


@pytest.mark.parametrize("lens", [(1,), (3, 1, 7), tuple(range(1, 33))])
def test_fast_pack_equals_checked(lens):
    rng = np.random.default_rng(len(lens))
    seqs = random_seqs(rng, lens)
    a = _pack_fast(seqs, 6, 35)
    b = _pack_checked(seqs, 6, 35)
    assert a is not None
    for x, y in ((a.steps, b.steps), (a.offsets, b.offsets), (a.ctx, b.ctx)):
        assert np.array_equal(x, y)
    assert a.max_steps == max(lens)


def test_integer_and_list_inputs_are_cast():
    seqs = [Seq(np.ones((2, 6), dtype=np.int32), list(range(35))), Seq(np.zeros((1, 6)), np.ones(35))]
    h = pack_sequences(seqs, 6, 35)
    assert h.steps.dtype == np.float64 and h.ctx.dtype == np.float64
    assert h.offsets.tolist() == [0, 2, 3]


@pytest.mark.parametrize("bad", [
    [Seq(np.ones((2, 5)), np.ones(35))],                      # step width
    [Seq(np.ones((2, 6)), np.ones(34))],                      # context length
    [Seq(np.ones((0, 6)), np.ones(35))],                      # empty program
    [Seq(np.ones(6), np.ones(35))],                           # 1-D steps
    [Seq(np.ones((2, 6)), np.ones(35)), Seq(np.ones((2, 6)), np.ones(36))],
    [Seq(np.ones((2, 6)), np.ones(35)), Seq(np.ones((2, 7)), np.ones(35))],
    [Seq(np.ones((2, 6)), np.ones(36)), Seq(np.ones((2, 6)), np.ones(34))],  # same total size
])
def test_malformed_input_raises(bad):
    with pytest.raises(DataValidationError):
        pack_sequences(bad, 6, 35)


def test_empty_batch_raises():
    with pytest.raises(DataValidationError):
        pack_sequences([], 6, 35)


def _native_pack(seqs, dtype, d0=6, C=35):
    out = {}

    def alloc(rows, n, w, c):
        out["s"], out["c"] = np.full((rows, w), np.nan, dtype), np.full((n, c), np.nan, dtype)
        return out["s"], out["c"]

    off = _pack_native(seqs, d0, C, alloc)
    return off, out


def test_native_packer_is_built():
    assert _native() is not None, "csrc/host/tt_pack.c was not built (paper_2304_05430_b200.build)"


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_native_pack_equals_checked(dtype):
    rng = np.random.default_rng(5)
    seqs = random_seqs(rng, list(rng.integers(1, 20, size=300)))
    # mixed input dtypes and non-contiguous views go through the strided copy
    seqs[3] = Seq(seqs[3].steps.astype(np.float32), seqs[3].context)
    big = np.asfortranarray(rng.normal(size=(4, 6)))
    seqs[7] = Seq(big, np.ascontiguousarray(rng.normal(size=70))[::2])
    off, out = _native_pack(seqs, dtype)
    want = _pack_checked(seqs, 6, 35)
    assert np.array_equal(off, want.offsets)
    assert np.array_equal(out["s"], want.steps.astype(dtype))
    assert np.array_equal(out["c"], want.ctx.astype(dtype))
    h = pack_sequences(seqs, 6, 35)
    assert np.array_equal(h.steps, want.steps) and np.array_equal(h.ctx, want.ctx)


def test_native_pack_infers_widths_and_declines_non_float():
    rng = np.random.default_rng(6)
    seqs = random_seqs(rng, [2, 3], d0=164)
    off, out = _native_pack(seqs, np.float64, d0=-1, C=-1)
    assert off.tolist() == [0, 2, 5] and out["s"].shape == (5, 164)
    ints = [Seq(np.ones((2, 6), dtype=np.int32), np.ones(35))]
    assert _native_pack(ints, np.float64)[0] is None  # numpy path casts these


@pytest.mark.parametrize("bad", [
    [Seq(np.ones((2, 5)), np.ones(35))],
    [Seq(np.ones((0, 6)), np.ones(35))],
    [Seq(np.ones(6), np.ones(35))],
    [Seq(np.ones((2, 6)), np.ones(35)), Seq(np.ones((2, 6)), np.ones(36))],
])
def test_native_pack_declines_malformed(bad):
    assert _native_pack(bad, np.float64)[0] is None
    with pytest.raises(DataValidationError):
        pack_sequences(bad, 6, 35)


def test_native_pack_rejects_bad_alloc():
    rng = np.random.default_rng(1)
    seqs = random_seqs(rng, [2, 2])
    with pytest.raises(ValueError):
        _pack_native(seqs, 6, 35, lambda r, n, w, c: (np.empty(1), np.empty(1)))
    with pytest.raises(RuntimeError):
        _pack_native(seqs, 6, 35, lambda r, n, w, c: (_ for _ in ()).throw(RuntimeError("x")))


def test_non_native_byte_order_and_unaligned_inputs_pack_correctly():
    """'>f8' arrays were memcpy'd as garbage by the native packer.
    Now it declines them (returns None) and the numpy path converts them."""
    rng = np.random.default_rng(8)
    seqs = random_seqs(rng, [3, 5, 2])
    swapped = [Seq(s.steps.astype(">f8"), s.context.astype(">f4")) for s in seqs]
    want = _pack_checked([Seq(s.steps, s.context.astype(np.float32)) for s in seqs], 6, 35)
    assert _native_pack(swapped, np.float64)[0] is None
    h = pack_sequences(swapped, 6, 35)
    assert np.array_equal(h.steps, want.steps) and np.array_equal(h.ctx, want.ctx)
    buf = np.zeros(3 * 6 * 8 + 1, dtype=np.uint8)
    una = np.frombuffer(buf.data, dtype=np.float64, count=18, offset=1).reshape(3, 6)
    assert not una.flags.aligned
    seqs2 = [Seq(np.ascontiguousarray(seqs[0].steps), seqs[0].context)]
    buf[1:1 + 18 * 8] = np.frombuffer(seqs2[0].steps.tobytes(), dtype=np.uint8)
    un_seqs = [Seq(una, seqs2[0].context)]
    assert _native_pack(un_seqs, np.float64)[0] is None
    h = pack_sequences(un_seqs, 6, 35)
    assert np.array_equal(h.steps, seqs2[0].steps)
