"""K9: program layout (replaces the padded batch of tuner.py:36-52 _pack).

The reference pads every chunk of 256 programs to (B, Tmax, 6) plus a mask;
padding is inert (masked steps hold state, -1e30 logits, masked mean), so the
device layout is CSR instead: all step rows of all programs back to back,
int64 row offsets, one context row per program.  A program's forward
direction runs t = 0..T-1 and its backward direction t = T-1..0 from zero
state, which equals the reference's reversed padded sequence
(tuner.py:242-243) exactly.

Inputs are duck-typed StepSequence objects (features.py:70-92): ``.steps``
(T, step_width) and ``.context`` (ctx_len,).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device
from .errors import DataValidationError


@dataclass
class HostPrograms:
    steps: np.ndarray    # (rows, d0) float64
    offsets: np.ndarray  # (n + 1,) int64
    ctx: np.ndarray      # (n, C) float64

    @property
    def n(self) -> int:
        return self.offsets.shape[0] - 1

    @property
    def max_steps(self) -> int:
        return int(np.max(np.diff(self.offsets))) if self.n else 0


def _native():
    try:
        from . import _ttpack
    except ImportError:  # not built: the vectorised numpy path below
        return None
    return _ttpack


def _pack_native(seqs, step_width, ctx_len, alloc):
    """csrc/host/tt_pack.c: one pass over the list (buffer protocol), dtype
    conversion while copying into the buffers ``alloc(rows, n, d0, C)``
    returns.  Returns the int64 offsets, or None (module missing / malformed
    item: the caller's numpy path reports the exact error)."""
    mod = _native()
    if mod is None or len(seqs) == 0:
        return None
    lens = mod.pack(seqs, -1 if step_width is None else int(step_width),
                    -1 if ctx_len is None else int(ctx_len), alloc)
    if lens is None:
        return None
    lens = np.frombuffer(lens, dtype=np.int64)
    off = np.zeros(lens.shape[0] + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return off


def pack_sequences(seqs, step_width: int | None = None, ctx_len: int | None = None) -> HostPrograms:
    if len(seqs) == 0:
        raise DataValidationError("empty sequence batch")
    out = {}

    def alloc(rows, n, d0, C):
        out["s"], out["c"] = np.empty((rows, d0)), np.empty((n, C))
        return out["s"], out["c"]

    off = _pack_native(seqs, step_width, ctx_len, alloc)
    if off is not None:
        return HostPrograms(out["s"], off, out["c"])
    fast = _pack_fast(seqs, step_width, ctx_len)
    if fast is not None:
        return fast
    return _pack_checked(seqs, step_width, ctx_len)


def _pack_fast(seqs, step_width, ctx_len) -> HostPrograms | None:
    """Vectorised packing for well-formed input (numpy does the shape checks);
    None sends malformed input to the per-item path for the exact message."""
    n = len(seqs)
    try:
        st = [s.steps for s in seqs]
        cx = [s.context for s in seqs]
        lens = np.fromiter(map(len, st), dtype=np.int64, count=n)
        clens = np.fromiter(map(len, cx), dtype=np.int64, count=n)
        steps = np.concatenate(st, axis=0, dtype=np.float64)
        ctx = np.concatenate(cx, axis=0, dtype=np.float64)
    except (ValueError, TypeError, AttributeError):
        return None
    C = int(clens[0])
    if (steps.ndim != 2 or ctx.ndim != 1 or lens.min() < 1 or steps.shape[0] != int(lens.sum())
            or np.any(clens != C) or ctx.shape[0] != n * C):
        return None
    ctx = ctx.reshape(n, C)
    if (step_width is not None and steps.shape[1] != step_width) or (
            ctx_len is not None and ctx.shape[1] != ctx_len):
        return None
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return HostPrograms(steps, off, ctx)


def _pack_checked(seqs, step_width, ctx_len) -> HostPrograms:
    steps = [np.asarray(s.steps, dtype=np.float64) for s in seqs]
    ctxs = [np.asarray(s.context, dtype=np.float64) for s in seqs]
    d0 = steps[0].shape[1] if steps[0].ndim == 2 else -1
    C = ctxs[0].shape[0] if ctxs[0].ndim == 1 else -1
    if step_width is not None and d0 != step_width:
        raise DataValidationError(f"steps must be (n, {step_width}), got {steps[0].shape}")
    if ctx_len is not None and C != ctx_len:
        raise DataValidationError(f"context must have {ctx_len} slots, got {ctxs[0].shape}")
    lens = np.empty(len(seqs), dtype=np.int64)
    for i, (st, cx) in enumerate(zip(steps, ctxs)):
        if st.ndim != 2 or st.shape[1] != d0 or st.shape[0] < 1:
            raise DataValidationError(f"steps must be (n >= 1, {d0}), got {st.shape}")
        if cx.shape != (C,):
            raise DataValidationError(f"context must have {C} slots, got {cx.shape}")
        lens[i] = st.shape[0]
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return HostPrograms(np.concatenate(steps, axis=0), off, np.stack(ctxs))


class DevicePrograms:
    """Device-resident CSR programs in the compute dtype."""

    def __init__(self, host: HostPrograms, precision: str = "fp32"):
        dt = _device.real_dtype(precision)
        self._set(precision, host.offsets, _device.to_dev(host.steps.reshape(-1), dt),
                  _device.to_dev(host.ctx.reshape(-1), dt), host.steps.shape[1], host.ctx.shape[1])

    def _set(self, precision, offsets, steps, ctx, d0, C):
        self.precision = precision
        self.n = offsets.shape[0] - 1
        self.d0, self.C = int(d0), int(C)
        self.max_steps = int(np.max(np.diff(offsets))) if self.n else 0
        self.steps, self.ctx = steps, ctx
        self.offsets = _device.to_dev(offsets.astype(np.int64))
        self.host_offsets = offsets

    @classmethod
    def from_sequences(cls, seqs, precision="fp32", step_width=None, ctx_len=None):
        """Host sequences -> device CSR.  With the native packer the rows are
        converted straight into pinned compute-dtype staging buffers and
        copied with one async H2D each (no float64 intermediate)."""
        if len(seqs) == 0:
            raise DataValidationError("empty sequence batch")
        t = _device.require_cuda()
        dt = _device.real_dtype(precision)
        out = {}

        def alloc(rows, n, d0, C):
            out["s"] = t.empty((rows, d0), dtype=dt, pin_memory=True)
            out["c"] = t.empty((n, C), dtype=dt, pin_memory=True)
            out["d0"], out["C"] = d0, C
            return out["s"].numpy(), out["c"].numpy()

        off = _pack_native(seqs, step_width, ctx_len, alloc)
        if off is None:
            return cls(pack_sequences(seqs, step_width, ctx_len), precision)
        dev = _device.device()
        self = cls.__new__(cls)
        self._set(precision, off, out["s"].reshape(-1).to(dev, non_blocking=True),
                  out["c"].reshape(-1).to(dev, non_blocking=True), out["d0"], out["C"])
        # (torch's pinned-host allocator holds the staging blocks until the
        # copies recorded on the current stream have completed)
        return self
