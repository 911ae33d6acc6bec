"""§8(f) row 1: batched featurization and labels (featurize.py) against the
reference's own encoders, bit-exact, including its error behaviour.  Needs
the reference package (build container); skipped on the GPU box."""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present (GPU box)")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from tensortune import benchmarks, features

    from paper_2304_05430_b200.featurize import make_encoders

    ds = benchmarks.pruning_benchmark(seed=1, n_tasks=24, records_per_task=60)
    return features, make_encoders(features), ds


def _same_seqs(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert type(x) is type(y)
        assert x.steps.tobytes() == y.steps.tobytes() and x.steps.shape == y.steps.shape
        assert x.context.tobytes() == y.context.tobytes()


def test_sequence_and_flat_batches_are_bit_exact(ref):
    features, (enc_seq, enc_flat), ds = ref
    ids = [r.record_id for r in ds.records if not r.error_flag]
    rng = np.random.default_rng(0)
    ids = [ids[i] for i in rng.permutation(len(ids))]  # any record order
    s1, y1 = features.encode_sequence_batch(ds, ids)
    s2, y2 = enc_seq(ds, ids)
    _same_seqs(s1, s2)
    assert y1.tobytes() == y2.tobytes()
    X1, z1 = features.encode_flat_batch(ds, ids)
    X2, z2 = enc_flat(ds, ids)
    assert X1.tobytes() == X2.tobytes() and z1.tobytes() == z2.tobytes()


def test_empty_batch(ref):
    features, (enc_seq, enc_flat), ds = ref
    s, y = enc_seq(ds, [])
    assert s == [] and y.shape == (0,)
    X, z = enc_flat(ds, [])
    a, b = features.encode_flat_batch(ds, [])
    assert X.shape == a.shape and z.shape == b.shape


def test_error_records_raise_like_reference(ref):
    features, (enc_seq, enc_flat), ds = ref
    bad = next(r.record_id for r in ds.records if r.error_flag)
    good = next(r.record_id for r in ds.records if not r.error_flag)
    for ours, theirs in ((enc_seq, features.encode_sequence_batch),
                         (enc_flat, features.encode_flat_batch)):
        with pytest.raises(features.DataValidationError) as e1:
            theirs(ds, [good, bad])
        with pytest.raises(features.DataValidationError) as e2:
            ours(ds, [good, bad])
        assert str(e1.value) == str(e2.value)
        with pytest.raises(KeyError):
            ours(ds, ["no-such-record"])


def test_unresolvable_task_and_tile_cap(ref):
    features, (enc_seq, enc_flat), ds = ref
    from tensortune.data import Dataset

    rec = next(r for r in ds.records if not r.error_flag)
    orphan = dataclasses.replace(rec, record_id="orphan", task_id="missing")
    wide = dataclasses.replace(rec, record_id="wide", schedule=dataclasses.replace(
        rec.schedule, tile_factors=((1,) * 5, (1,) * 5)))
    ds2 = Dataset.__new__(Dataset)
    ds2.__dict__.update(ds.__dict__)
    ds2.record_by_id = dict(ds.record_by_id, orphan=orphan, wide=wide)
    for ids in (["orphan"], ["wide"]):
        for ours, theirs in ((enc_seq, features.encode_sequence_batch),
                             (enc_flat, features.encode_flat_batch)):
            try:
                want = theirs(ds2, ids)
            except Exception as e:  # noqa: BLE001
                with pytest.raises(Exception) as got:
                    ours(ds2, ids)
                assert str(got.value) == str(e)
            else:
                got = ours(ds2, ids)
                if isinstance(want[0], list):
                    _same_seqs(want[0], got[0])
                else:
                    assert want[0].tobytes() == got[0].tobytes()
                assert want[1].tobytes() == got[1].tobytes()
