"""fp32 tensor-core tuner scorer (tt_tuner_predict_f32tc) against the fp64
kernel and the fp32 CUDA-core kernel on the bench's 262,144 programs:
max |error| vs fp64, programs/s, small-batch latency and launch-size
invariance.  Prints JSON lines.

    python tools/x3_probe.py
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2304_05430_b200 import RecurrentAttentionTuner, _device, _lib  # noqa: E402
from paper_2304_05430_b200.layout import DevicePrograms, HostPrograms  # noqa: E402


def f32tc(est, prog, dims, flat):
    lib = _lib.load()
    nbytes = lib.tt_tuner_predict_f32tc_workspace_bytes(dims["L"], dims["H"], prog.max_steps, prog.n)
    ws = _device.workspace(nbytes, "x3probe")
    out = torch.empty(prog.n, dtype=torch.float32, device="cuda")
    _lib.call("tt_tuner_predict_f32tc", flat.data_ptr(), prog.steps.data_ptr(), prog.offsets.data_ptr(),
              prog.ctx.data_ptr(), prog.n, dims["L"], dims["H"], dims["heads"], dims["U"], dims["d0"],
              dims["C"], prog.max_steps, out.data_ptr(), ws.data_ptr(), nbytes, _device.stream_ptr())
    return out


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return out, float(np.median(ts))


def main():
    st, of, cx, y, ln = bench.synth(seed=0)
    hp = HostPrograms(st, of, cx)
    est = RecurrentAttentionTuner(seed=0)
    est._init_params()
    dims = est._dims()
    est.precision = "fp64"
    p64 = DevicePrograms(hp, "fp64")
    ref = est._predict_programs(p64, dims).cpu().numpy()
    est.precision = "fp32_cuda"
    prog = DevicePrograms(hp, "fp32")
    flat = est._dev_params(dims)
    o32, t32 = timed(lambda: est._predict_programs(prog, dims, flat))
    otc, ttc = timed(lambda: f32tc(est, prog, dims, flat))
    o32, otc = o32.cpu().numpy().astype(np.float64), otc.cpu().numpy().astype(np.float64)
    print(json.dumps({"n": prog.n, "fp32_cuda_err": float(np.abs(o32 - ref).max()),
                      "f32tc_err": float(np.abs(otc - ref).max()),
                      "f32tc_mean_err": float(np.abs(otc - ref).mean()),
                      "fp32_cuda_per_s": prog.n / t32, "f32tc_per_s": prog.n / ttc}), flush=True)
    if "--phases" in sys.argv:
        if "--n1" in sys.argv:  # one program: the latency of a single-tile call
            prog = DevicePrograms(HostPrograms(st[: of[1]], of[:2], cx[:1]), "fp32")
        f32tc(est, prog, dims, flat)
        torch.cuda.synchronize()
        buf = np.zeros(30, dtype=np.int64)
        _lib.call("tt_debug_x3_phase_times", buf.ctypes.data, 30)
        names = ["d_full", "x_arrived", "gates_loaded", "act_done", "h_arrived", "mma_x_ready", "-",
                 "mma_h_ready", "mma_committed"]
        t0 = buf[0]
        print(json.dumps({f"s{2 + i // 9}_{names[i % 9]}": int(buf[i] - t0) for i in range(18) if i % 9 != 6}))
        ld = {f"ld{k // 2}_{'start' if k % 2 == 0 else 'mma_done'}": int(buf[18 + k] - buf[18]) for k in range(12)}
        print(json.dumps(ld))
    if "--fixed" in sys.argv:  # per-call time at uniform program lengths
        m = 4 * 148 * 128
        for T in (1, 2, 4, 7, 10):
            off = np.arange(0, (m + 1) * T, T, dtype=np.int64)
            hpf = HostPrograms(np.resize(st, (m * T, st.shape[1])), off, np.resize(cx, (m, cx.shape[1])))
            pf = DevicePrograms(hpf, "fp32")
            _, t = timed(lambda: f32tc(est, pf, dims, flat))
            print(json.dumps({"T": T, "programs": m, "us_per_call": t * 1e6}), flush=True)
    if "--quick" in sys.argv or "--phases" in sys.argv or "--fixed" in sys.argv:
        return
    # launch-size invariance and small-batch latency
    for m in (1, 8, 100, 148, 149, 1000, 20000):
        sub = DevicePrograms(HostPrograms(st[: of[m]], of[: m + 1], cx[:m]), "fp32")
        o, t = timed(lambda: f32tc(est, sub, dims, flat))
        oc, tc = timed(lambda: est._predict_programs(sub, dims, flat))
        o = o.cpu().numpy().astype(np.float64)
        print(json.dumps({"n": m, "bit_equal_to_full_batch": bool(np.array_equal(o, otc[:m])),
                          "f32tc_us": t * 1e6, "fp32_cuda_us": tc * 1e6}), flush=True)


if __name__ == "__main__":
    main()
