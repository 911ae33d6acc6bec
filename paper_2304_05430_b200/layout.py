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


def pack_sequences(seqs, step_width: int | None = None, ctx_len: int | None = None,
                   min_steps: int = 1) -> HostPrograms:
    if len(seqs) == 0:
        raise DataValidationError("empty sequence batch")
    out = {}

    def alloc(rows, n, d0, C):
        out["s"], out["c"] = np.empty((rows, d0)), np.empty((n, C))
        return out["s"], out["c"]

    off = _pack_native(seqs, step_width, ctx_len, alloc)
    if off is not None:
        return HostPrograms(out["s"], off, out["c"])
    fast = _pack_fast(seqs, step_width, ctx_len, min_steps)
    if fast is not None:
        return fast
    return _pack_checked(seqs, step_width, ctx_len, min_steps)


def _pack_fast(seqs, step_width, ctx_len, min_steps=1) -> HostPrograms | None:
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
    if (steps.ndim != 2 or ctx.ndim != 1 or lens.min() < min_steps or steps.shape[0] != int(lens.sum())
            or np.any(clens != C) or ctx.shape[0] != n * C):
        return None
    ctx = ctx.reshape(n, C)
    if (step_width is not None and steps.shape[1] != step_width) or (
            ctx_len is not None and ctx.shape[1] != ctx_len):
        return None
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    return HostPrograms(steps, off, ctx)


def _pack_checked(seqs, step_width, ctx_len, min_steps=1) -> HostPrograms:
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
        if st.ndim != 2 or st.shape[1] != d0 or st.shape[0] < min_steps:
            raise DataValidationError(f"steps must be (n >= {min_steps}, {d0}), got {st.shape}")
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
    def from_sequences(cls, seqs, precision="fp32", step_width=None, ctx_len=None, min_steps=1):
        """Host sequences -> device CSR.  With the native packer the rows are
        converted straight into ONE pinned staging buffer [steps | ctx |
        offsets] in the compute dtype and uploaded with one async copy."""
        if len(seqs) == 0:
            raise DataValidationError("empty sequence batch")
        t = _device.require_cuda()
        dt = _device.real_dtype(precision)
        esz = 8 if dt == t.float64 else 4
        npdt = np.float64 if esz == 8 else np.float32
        out = {}

        def alloc(rows, n, d0, C):
            ns, nc = rows * d0, n * C
            o_c = -(-ns * esz // 16) * 16
            o_o = -(-(o_c + nc * esz) // 16) * 16
            buf = t.empty(o_o + (n + 1) * 8, dtype=t.uint8, pin_memory=True)
            hb = buf.numpy()
            out.update(buf=buf, hb=hb, d0=d0, C=C, ns=ns, nc=nc, o_c=o_c, o_o=o_o)
            return hb[:ns * esz].view(npdt), hb[o_c:o_c + nc * esz].view(npdt)

        off = _pack_native(seqs, step_width, ctx_len, alloc)
        if off is None:  # malformed input, or programs without steps (predict)
            return cls(pack_sequences(seqs, step_width, ctx_len, min_steps), precision)
        o = out
        o["hb"][o["o_o"]:].view(np.int64)[:] = off
        dev = o["buf"].to(_device.device(), non_blocking=True)
        # (torch's pinned-host allocator keeps the staging block until the
        # copy recorded on the current stream has completed)
        self = cls.__new__(cls)
        self.precision = precision
        self.n = off.shape[0] - 1
        self.d0, self.C = int(o["d0"]), int(o["C"])
        self.max_steps = int(np.max(np.diff(off)))
        self.steps = dev[:o["ns"] * esz].view(dt)
        self.ctx = dev[o["o_c"]:o["o_c"] + o["nc"] * esz].view(dt)
        self.offsets = dev[o["o_o"]:].view(t.int64)
        self.host_offsets = off
        return self
