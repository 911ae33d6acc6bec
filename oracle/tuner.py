"""RecurrentAttentionTuner restated (TEST INFRASTRUCTURE ONLY).

Source: /root/reference/pkg/src/tensortune/estimators/tuner.py
  init            :181-211  Glorot from default_rng(seed), dict order, forget bias 1
  pack            :36-52    pad to (B, Tmax, d0) + {0,1} mask + ctx
  lstm direction  :61-151   gate blocks [i|f|g|o], masked steps hold h and c
  stack           :233-246  bw = forward over the reversed padded batch
  attention       :248-274  masked mean p0, K/V without bias, U passes of
                            nh-head softmax pooling (scale before -1e30 mask)
  head            :276-279  tanh(z W1 + b1) W2 + b2 -> logistic, z=[pooled|ctx]
  backward        :287-360
  loss            :364-376  ranking on the sigmoid output or MSE
  train loop      :427-466  default_rng(seed + offset).permutation per epoch
  predict         :468-476  chunks of 256

Everything is float64 numpy over a padded batch, i.e. the same cost profile
as the reference, so this module doubles as the CPU baseline in bench.py.
"""

from __future__ import annotations

import numpy as np

from .adam import AdamOracle
from .losses import loss_and_dscore
from .metrics import grouped_pca
from .mlp import glorot

HEAD_HIDDEN = 64


# -- parameters ---------------------------------------------------------------


def init_params(seed: int, layers: int = 3, hidden: int = 32, d0: int = 6,
                ctx_len: int = 35) -> dict:
    rng = np.random.default_rng(seed)
    H, D = hidden, 2 * hidden
    p: dict = {}
    for l in range(layers):
        fan_in = d0 if l == 0 else D
        for side in ("fw", "bw"):
            key = f"lstm{l}_{side}"
            p[key + "_Wx"] = glorot(rng, fan_in, 4 * H)
            p[key + "_Wh"] = glorot(rng, H, 4 * H)
            bias = np.zeros(4 * H)
            bias[H : 2 * H] = 1.0
            p[key + "_b"] = bias
    for m in ("Wq", "Wk", "Wv", "Wo"):
        p["attn_" + m] = glorot(rng, D, D)
    p["attn_bq"] = np.zeros(D)
    p["attn_bo"] = np.zeros(D)
    p["head_W1"] = glorot(rng, D + ctx_len, HEAD_HIDDEN)
    p["head_b1"] = np.zeros(HEAD_HIDDEN)
    p["head_W2"] = glorot(rng, HEAD_HIDDEN, 1)
    p["head_b2"] = np.zeros(1)
    return p


def n_layers(p: dict) -> int:
    return sum(1 for k in p if k.endswith("_fw_Wh"))


def hidden_of(p: dict) -> int:
    return p["lstm0_fw_Wh"].shape[0]


def groups(p: dict) -> dict:
    out = {"recurrent": [], "attention": [], "head": []}
    for k in p:
        g = "recurrent" if k.startswith("lstm") else "attention" if k.startswith("attn") else "head"
        out[g].append(k)
    return out


# -- layout -------------------------------------------------------------------


def pack(seqs):
    """Zero-padded (B, Tmax, d0) steps, (B, Tmax) mask, (B, C) contexts."""
    lens = [s.steps.shape[0] for s in seqs]
    d0 = seqs[0].steps.shape[1]
    C = seqs[0].context.shape[0]
    B, T = len(seqs), max(lens)
    X = np.zeros((B, T, d0))
    M = np.zeros((B, T))
    Z = np.zeros((B, C))
    for b, s in enumerate(seqs):
        X[b, : lens[b]] = s.steps
        M[b, : lens[b]] = 1.0
        Z[b] = s.context
    return X, M, Z


def _logistic(x):
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


# -- one LSTM direction ---------------------------------------------------------


def _dir_forward(Wx, Wh, b, X, M):
    B, T, _ = X.shape
    H = Wh.shape[0]
    proj = (X.reshape(B * T, -1) @ Wx).reshape(B, T, 4 * H)
    h = np.zeros((B, H))
    c = np.zeros((B, H))
    out = np.empty((B, T, H))
    keep = {k: np.empty((B, T, H)) for k in ("i", "f", "g", "o", "tc", "hp", "cp")}
    for t in range(T):
        z = proj[:, t] + h @ Wh + b
        i = _logistic(z[:, :H])
        f = _logistic(z[:, H : 2 * H])
        g = np.tanh(z[:, 2 * H : 3 * H])
        o = _logistic(z[:, 3 * H :])
        cn = f * c + i * g
        tc = np.tanh(cn)
        hn = o * tc
        for k, v in (("i", i), ("f", f), ("g", g), ("o", o), ("tc", tc), ("hp", h), ("cp", c)):
            keep[k][:, t] = v
        m = M[:, t][:, None]
        c = m * cn + (1.0 - m) * c
        h = m * hn + (1.0 - m) * h
        out[:, t] = h
    keep["X"], keep["M"] = X, M
    return out, keep


def _dir_backward(Wx, Wh, keep, d_out):
    X, M = keep["X"], keep["M"]
    B, T, _ = X.shape
    H = Wh.shape[0]
    dproj = np.zeros((B, T, 4 * H))
    dWh = np.zeros_like(Wh)
    db = np.zeros(4 * H)
    dh = np.zeros((B, H))
    dc = np.zeros((B, H))
    for t in reversed(range(T)):
        m = M[:, t][:, None]
        i, f, g, o = keep["i"][:, t], keep["f"][:, t], keep["g"][:, t], keep["o"][:, t]
        tc, hp, cp = keep["tc"][:, t], keep["hp"][:, t], keep["cp"][:, t]
        dh_all = d_out[:, t] + dh
        dh_live, dh_pass = dh_all * m, dh_all * (1.0 - m)
        dc_live, dc_pass = dc * m, dc * (1.0 - m)
        do = dh_live * tc
        dc_live = dc_live + dh_live * o * (1.0 - tc**2)
        dz = np.concatenate(
            [
                dc_live * g * i * (1.0 - i),
                dc_live * cp * f * (1.0 - f),
                dc_live * i * (1.0 - g**2),
                do * o * (1.0 - o),
            ],
            axis=1,
        )
        dc = dc_live * f + dc_pass
        dproj[:, t] = dz
        dWh += hp.T @ dz
        db += dz.sum(axis=0)
        dh = dz @ Wh.T + dh_pass
    flat = dproj.reshape(B * T, -1)
    dWx = X.reshape(B * T, -1).T @ flat
    dX = (flat @ Wx.T).reshape(X.shape)
    return dX, dWx, dWh, db


# -- full model -----------------------------------------------------------------


def forward(p: dict, X, M, Z, heads: int = 2, unroll: int = 2):
    L = n_layers(p)
    H = hidden_of(p)
    D = 2 * H
    dh = D // heads
    cur = X
    layer_keep = []
    for l in range(L):
        a = f"lstm{l}_fw"
        r = f"lstm{l}_bw"
        o_f, k_f = _dir_forward(p[a + "_Wx"], p[a + "_Wh"], p[a + "_b"], cur, M)
        o_b, k_b = _dir_forward(p[r + "_Wx"], p[r + "_Wh"], p[r + "_b"], cur[:, ::-1], M[:, ::-1])
        layer_keep.append((k_f, k_b))
        cur = np.concatenate([o_f, o_b[:, ::-1]], axis=2)
    S = cur
    B, T, _ = S.shape
    cnt = np.maximum(M.sum(axis=1, keepdims=True), 1.0)
    p0 = (S * M[:, :, None]).sum(axis=1) / cnt
    Kh = (S.reshape(B * T, D) @ p["attn_Wk"]).reshape(B, T, heads, dh).transpose(0, 2, 1, 3)
    Vh = (S.reshape(B * T, D) @ p["attn_Wv"]).reshape(B, T, heads, dh).transpose(0, 2, 1, 3)
    bias = np.where(M[:, None, :] > 0, 0.0, -1e30)
    pooled = p0
    passes = []
    for _ in range(unroll):
        q = (pooled @ p["attn_Wq"] + p["attn_bq"]).reshape(B, heads, dh)
        lg = np.einsum("bhd,bhtd->bht", q, Kh) / np.sqrt(dh) + bias
        lg = lg - lg.max(axis=2, keepdims=True)
        w = np.exp(lg)
        a = w / w.sum(axis=2, keepdims=True)
        mix = np.einsum("bht,bhtd->bhd", a, Vh).reshape(B, D)
        passes.append((pooled, q, a, mix))
        pooled = mix @ p["attn_Wo"] + p["attn_bo"]
    z = np.concatenate([pooled, Z], axis=1)
    a1 = np.tanh(z @ p["head_W1"] + p["head_b1"])
    yhat = _logistic((a1 @ p["head_W2"] + p["head_b2"])[:, 0])
    cache = dict(layers=layer_keep, S=S, K=Kh, V=Vh, cnt=cnt, M=M, passes=passes,
                 z=z, a1=a1, yhat=yhat, heads=heads)
    return yhat, cache


def backward(p: dict, cache: dict, d_y) -> dict:
    L = n_layers(p)
    H = hidden_of(p)
    D = 2 * H
    heads = cache["heads"]
    dh = D // heads
    S, Kh, Vh, M = cache["S"], cache["K"], cache["V"], cache["M"]
    B, T, _ = S.shape
    g = {k: np.zeros_like(v) for k, v in p.items()}
    yhat = cache["yhat"]
    dl = (d_y * yhat * (1.0 - yhat))[:, None]
    g["head_W2"] = cache["a1"].T @ dl
    g["head_b2"] = dl.sum(axis=0)
    da1 = (dl @ p["head_W2"].T) * (1.0 - cache["a1"] ** 2)
    g["head_W1"] = cache["z"].T @ da1
    g["head_b1"] = da1.sum(axis=0)
    dpool = (da1 @ p["head_W1"].T)[:, :D]
    dK = np.zeros_like(Kh)
    dV = np.zeros_like(Vh)
    scale = 1.0 / np.sqrt(dh)
    for p_in, q, a, mix in reversed(cache["passes"]):
        g["attn_Wo"] += mix.T @ dpool
        g["attn_bo"] += dpool.sum(axis=0)
        dmix = (dpool @ p["attn_Wo"].T).reshape(B, heads, dh)
        da = np.einsum("bhd,bhtd->bht", dmix, Vh)
        dV += np.einsum("bht,bhd->bhtd", a, dmix)
        dlg = a * (da - (da * a).sum(axis=2, keepdims=True))
        dq = (np.einsum("bht,bhtd->bhd", dlg, Kh) * scale).reshape(B, D)
        dK += np.einsum("bht,bhd->bhtd", dlg, q) * scale
        g["attn_Wq"] += p_in.T @ dq
        g["attn_bq"] += dq.sum(axis=0)
        dpool = dq @ p["attn_Wq"].T
    dS = (dpool / cache["cnt"])[:, None, :] * M[:, :, None]
    dKf = dK.transpose(0, 2, 1, 3).reshape(B * T, D)
    dVf = dV.transpose(0, 2, 1, 3).reshape(B * T, D)
    Sf = S.reshape(B * T, D)
    g["attn_Wk"] += Sf.T @ dKf
    g["attn_Wv"] += Sf.T @ dVf
    dS = dS + (dKf @ p["attn_Wk"].T + dVf @ p["attn_Wv"].T).reshape(B, T, D)
    for l in reversed(range(L)):
        k_f, k_b = cache["layers"][l]
        a = f"lstm{l}_fw"
        r = f"lstm{l}_bw"
        dXf, g[a + "_Wx"], g[a + "_Wh"], g[a + "_b"] = _dir_backward(
            p[a + "_Wx"], p[a + "_Wh"], k_f, dS[:, :, :H])
        dXb, g[r + "_Wx"], g[r + "_Wh"], g[r + "_b"] = _dir_backward(
            p[r + "_Wx"], p[r + "_Wh"], k_b, dS[:, ::-1, H:])
        dS = dXf + dXb[:, ::-1]
    return g


def loss_and_gradients(p, seqs, y, kind="rmse", heads=2, unroll=2):
    X, M, Z = pack(seqs)
    yhat, cache = forward(p, X, M, Z, heads, unroll)
    loss, d = loss_and_dscore(kind, np.asarray(y, dtype=np.float64), yhat)
    return loss, backward(p, cache, d)


def predict(p, seqs, chunk=256, heads=2, unroll=2) -> np.ndarray:
    parts = []
    for lo in range(0, len(seqs), chunk):
        X, M, Z = pack(seqs[lo : lo + chunk])
        parts.append(forward(p, X, M, Z, heads, unroll)[0])
    return np.concatenate(parts) if parts else np.zeros(0)


def train(p, seqs, y, *, epochs, lr, batch_size=16, seed=0, seed_offset=1,
          trainable=None, eval_set=None, eval_groups=None, loss="rmse",
          heads=2, unroll=2):
    """The _train loop (tuner.py:427-466); mutates p, returns the curve."""
    y = np.asarray(y, dtype=np.float64)
    opt = AdamOracle(p, lr)
    rng = np.random.default_rng(seed + seed_offset)
    n = len(seqs)
    curve = []
    for epoch in range(epochs):
        order = rng.permutation(n)
        for lo in range(0, n, batch_size):
            b = order[lo : lo + batch_size]
            val, g = loss_and_gradients(p, [seqs[i] for i in b], y[b], loss, heads, unroll)
            if not np.isfinite(val):
                raise FloatingPointError(f"loss became non-finite at epoch {epoch}")
            if trainable is not None:
                g = {k: v for k, v in g.items() if k in trainable}
            opt.step(g)
        tr = float(np.sqrt(np.mean((predict(p, seqs, heads=heads, unroll=unroll) - y) ** 2)))
        va = vp = None
        if eval_set is not None:
            pv = predict(p, eval_set[0], heads=heads, unroll=unroll)
            yv = np.asarray(eval_set[1], dtype=np.float64)
            va = float(np.sqrt(np.mean((pv - yv) ** 2)))
            if eval_groups is not None:
                vp = grouped_pca(yv, pv, eval_groups)
        curve.append((tr, va, vp))
    return curve
