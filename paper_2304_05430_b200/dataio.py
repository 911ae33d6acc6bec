"""Dataset I/O <- data.py:507-657 (tensortune.v1 JSONL).

``loads_dataset`` / ``load_dataset`` / ``dumps_dataset`` / ``save_dataset``
with the reference's signatures, results and errors; the per-record work --
the bulk of a dataset file -- goes through the native codec
csrc/host/tt_jsonl.c (``_ttjsonl``):

* reading: the header, hardware and task lines are parsed by the
  reference's own ``loads_dataset`` (a few lines); the record lines by
  ``_ttjsonl.parse_records``, which builds the reference's own
  ``ScheduleConfig`` / ``MeasurementRecord`` dataclasses with the values
  ``from_json`` would give; then the reference's ``Dataset.build`` validates
  as usual.  Any line outside the canonical shape the writer produces (other
  key order, escapes, whitespace, unknown or missing fields, interleaved
  lines) -- and ``lenient=True`` -- sends the WHOLE text through the
  reference's reader, so results and error messages are the reference's.
* writing: the record lines come from ``_ttjsonl.dump_records`` (json.dumps
  spacing, ``format_cost`` for the cost); the output is byte-identical to the
  reference's ``dumps_dataset`` (tests/test_dataio.py), and any record the
  codec cannot render exactly (non-ASCII ids, the cost sentinel) falls back
  to the reference writer.

``install()`` patches these names into ``tensortune.data`` (and the modules
that imported them), so the CLI and every workflow read and write through
them.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

_REF: dict = {}


def _native():
    try:
        from . import _ttjsonl
    except ImportError:  # not built
        return None
    return _ttjsonl


def bind_reference() -> None:
    """Capture the reference's own reader/writer before install() patches them."""
    data = sys.modules["tensortune.data"]
    for name in ("loads_dataset", "dumps_dataset"):
        fn = getattr(data, name)
        if _REF.get(name) is None and getattr(fn, "__module__", "") != __name__:
            _REF[name] = fn


def _ref(name):
    bind_reference()
    return _REF[name]


_RECORD_PREFIX = b'{"type": "record"'


def loads_dataset(text: str, lenient: bool = False):
    data = sys.modules["tensortune.data"]
    mod = _native()
    if lenient or mod is None:
        return _ref("loads_dataset")(text, lenient=lenient)
    raw = text.encode("utf-8")
    first = raw.find(b"\n" + _RECORD_PREFIX)
    if first < 0:  # no records (or none in canonical form): the reference reads it all
        return _ref("loads_dataset")(text)
    try:
        pre = _ref("loads_dataset")(raw[:first + 1].decode("utf-8"))
    except data.DataValidationError:
        return _ref("loads_dataset")(text)  # the reference reports the first error itself
    if pre.records:  # a record line before the first canonical one: not the writer's layout
        return _ref("loads_dataset")(text)
    recs = mod.parse_records(raw, first + 1, len(raw), data.ScheduleConfig, data.MeasurementRecord)
    if recs is None:
        return _ref("loads_dataset")(text)
    return data.Dataset.build(list(pre.hardware), list(pre.tasks), recs)


def load_dataset(path, lenient: bool = False):
    return loads_dataset(Path(path).read_text(encoding="utf-8"), lenient=lenient)


def dumps_dataset(ds) -> str:
    data = sys.modules["tensortune.data"]
    mod = _native()
    body = mod.dump_records(ds.records) if mod is not None else None
    if body is None:
        return _ref("dumps_dataset")(ds)
    sep = (", ", ": ")
    lines = [json.dumps({"format": data.FORMAT_TAG}, separators=sep)]
    lines += [json.dumps({"type": "hardware", **hw.to_json()}, separators=sep) for hw in ds.hardware]
    lines += [json.dumps(task.to_json(), separators=sep) for task in ds.tasks]
    return "\n".join(lines) + "\n" + body


def save_dataset(ds, path) -> None:
    Path(path).write_text(dumps_dataset(ds), encoding="utf-8")
