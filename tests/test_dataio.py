"""Dataset I/O (paper_2304_05430_b200.dataio + the native record
codec csrc/host/tt_jsonl.c) against the reference's own reader and writer
(data.py:507-657): byte-identical text, equal datasets, identical errors."""

from __future__ import annotations

import os
import sys

import pytest

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = next((p for p in ("/root/reference/pkg/src", os.path.join(_ROOT, "baseline", "_ref"))
            if os.path.isdir(os.path.join(p, "tensortune"))), "")


@pytest.fixture(scope="module")
def ref():
    if not REF:
        pytest.skip("reference package not present")
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import tensortune.data as data
    from tensortune.benchmarks import pruning_benchmark, transfer_benchmark

    from paper_2304_05430_b200 import dataio

    dataio.bind_reference()
    assert dataio._native() is not None, "csrc/host/tt_jsonl.c was not built"
    ds1 = pruning_benchmark(seed=0, n_tasks=12, records_per_task=30)  # error records, CPU + GPU targets
    ds2 = transfer_benchmark(seed=1)[0]
    return data, dataio, (ds1, ds2)


def test_writer_is_byte_identical_and_reader_round_trips(ref):
    data, dataio, dss = ref
    for ds in dss:
        want = data.dumps_dataset(ds)
        got = dataio.dumps_dataset(ds)
        assert got == want
        back = dataio.loads_dataset(want)
        assert back == data.loads_dataset(want)
        assert back == ds
        assert dataio.dumps_dataset(back) == want
        # the fast path really ran: record objects are the reference's classes
        assert type(back.records[0]) is data.MeasurementRecord
        assert type(back.records[0].schedule) is data.ScheduleConfig


def test_thread_binding_error_records_and_cost_formats(ref):
    data, dataio, (ds, _) = ref
    recs = list(ds.records)
    assert any(r.error_flag for r in recs) and any(r.schedule.thread_binding for r in recs)
    # costs with few significant digits take format_cost's "%.8e" branch
    from dataclasses import replace

    recs[0] = replace(recs[0], mean_cost=1e-06) if not recs[0].error_flag else recs[0]
    recs[1] = replace(recs[1], mean_cost=0.5) if not recs[1].error_flag else recs[1]
    ds2 = data.Dataset.build(ds.hardware, ds.tasks, recs)
    assert dataio.dumps_dataset(ds2) == data.dumps_dataset(ds2)
    assert dataio.loads_dataset(data.dumps_dataset(ds2)) == ds2


def test_non_canonical_text_falls_back_with_the_references_errors(ref):
    data, dataio, (ds, _) = ref
    text = data.dumps_dataset(ds)
    lines = text.splitlines()
    i = next(k for k, ln in enumerate(lines) if '"type": "record"' in ln)
    variants = {
        "reordered keys": lines[:i] + [lines[i].replace('{"type": "record", ', '{') [:-1]
                                       + ', "type": "record"}'] + lines[i + 1:],
        "unknown field": lines[:i] + [lines[i][:-1] + ', "extra": 1}'] + lines[i + 1:],
        "blank line": lines[:i + 1] + [""] + lines[i + 1:],
        "bad json": lines[:i] + [lines[i][:-1]] + lines[i + 1:],
        "compact separators": lines[:i] + [lines[i].replace(", ", ",")] + lines[i + 1:],
        "float flops": lines[:i] + [lines[i].replace('"measured_flops": ', '"measured_flops": 1.5e1 + ')
                                    .replace(" + ", "")] + lines[i + 1:],
        "float flops small": lines[:i] + [lines[i].replace('"measured_flops": ', '"measured_flops": 0.0, "x": ')]
        + lines[i + 1:],
        "escaped id": lines[:i] + [lines[i].replace('"record_id": "', '"record_id": "\\u00e9')] + lines[i + 1:],
    }
    for name, ls in variants.items():
        t = "\n".join(ls) + "\n"
        try:
            want = data.loads_dataset(t)
        except Exception as exc:  # noqa: BLE001 - whatever the reference raises, we raise
            with pytest.raises(type(exc)) as got:
                dataio.loads_dataset(t)
            assert str(got.value) == str(exc), name
        else:
            assert dataio.loads_dataset(t) == want, name
    assert dataio.loads_dataset(text, lenient=True) == data.loads_dataset(text, lenient=True)


def test_ids_the_codec_cannot_render_fall_back_to_the_reference_writer(ref):
    data, dataio, (ds, _) = ref
    from dataclasses import replace

    recs = list(ds.records)
    recs[0] = replace(recs[0], record_id='r-"quoted"-é')
    ds2 = data.Dataset.build(ds.hardware, ds.tasks, recs)
    assert dataio.dumps_dataset(ds2) == data.dumps_dataset(ds2)
    assert dataio.loads_dataset(data.dumps_dataset(ds2)) == ds2
    recs[0] = replace(recs[0], record_id="@@MEAN-COST-SENTINEL@@")
    ds3 = data.Dataset.build(ds.hardware, ds.tasks, recs)
    with pytest.raises(data.DataValidationError, match="sentinel"):
        data.dumps_dataset(ds3)
    with pytest.raises(data.DataValidationError, match="sentinel"):
        dataio.dumps_dataset(ds3)


def test_empty_and_record_free_datasets(ref):
    data, dataio, (ds, _) = ref
    empty = data.Dataset.build(ds.hardware, ds.tasks, [])
    assert dataio.dumps_dataset(empty) == data.dumps_dataset(empty)
    assert dataio.loads_dataset(data.dumps_dataset(empty)) == empty
    with pytest.raises(data.DataValidationError, match="line 1"):
        dataio.loads_dataset("")


def test_cost_formatting_fuzz(ref):
    """format_cost's two branches over random magnitudes and digit counts."""
    import numpy as np
    from dataclasses import replace

    data, dataio, (ds, _) = ref
    rng = np.random.default_rng(0)
    good = [r for r in ds.records if not r.error_flag]
    costs = list(10.0 ** rng.uniform(-12, 3, size=len(good)))
    costs[:40] = [float(f"{c:.{k}g}") for c, k in zip(costs[:40], rng.integers(1, 10, size=40))]
    costs[40:44] = [5e-324, 1e-310, 1.0, 2.0 ** -1074 * 3]
    recs = [replace(r, mean_cost=float(c)) for r, c in zip(good, costs)]
    ds2 = data.Dataset.build(ds.hardware, ds.tasks, recs, validate=False)
    want = data.dumps_dataset(ds2)
    assert dataio.dumps_dataset(ds2) == want
    mod = dataio._native()
    raw = want.encode()
    first = raw.find(b'\n{"type": "record"') + 1
    parsed = mod.parse_records(raw, first, len(raw), data.ScheduleConfig, data.MeasurementRecord)
    assert [r.mean_cost for r in parsed] == [r.mean_cost for r in recs]
