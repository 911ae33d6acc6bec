"""K9 packing (layout.py): the vectorised path equals the per-item checked
path, and malformed input raises the reference's DataValidationError
(tuner.py:36-52 / features.py:70-92 shapes)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import Seq, random_seqs
from paper_2304_05430_b200.errors import DataValidationError
from paper_2304_05430_b200.layout import _pack_checked, _pack_fast, pack_sequences


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
