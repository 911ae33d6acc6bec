"""Pin the CPU oracle to the reference's own outputs (committed golden vectors).

Runs on CPU.  If any of these fail, the oracle -- and every GPU parity claim
built on it -- is unpinned.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, segments, unpack_seqs
from oracle import adam as oadam
from oracle import losses as oloss
from oracle import metrics as om
from oracle import mlp as omlp
from oracle import sampling as osamp
from oracle import tuner as otuner


def test_pca_matches_reference_exactly():
    g = golden("pca.npz")
    for (y, s), want in zip(segments(g["y"], g["s"], g["offsets"]), g["pca"]):
        assert om.pca(y, s) == want
    # brute force on the small ones (definition-level check of the golden set)
    for (y, s), want in list(zip(segments(g["y"], g["s"], g["offsets"]), g["pca"]))[:200]:
        assert om.brute_force_pca(y, s) == want


def test_topk_matches_reference_exactly():
    g = golden("topk.npz")
    for (y, s), t1, t5 in zip(segments(g["y"], g["s"], g["offsets"]), g["top1"], g["top5"]):
        assert om.top_k(y, s, 1) == t1
        assert om.top_k(y, s, min(5, len(y))) == t5


def test_ranking_grad_matches_reference():
    g = golden("ranking.npz")
    grads = []
    for (y, s), want in zip(segments(g["y"], g["s"], g["offsets"]), g["loss"]):
        l, d = oloss.pairwise_logistic(y, s)
        assert l == pytest.approx(want, rel=1e-13, abs=0)
        grads.append(d)
    np.testing.assert_allclose(np.concatenate(grads), g["grad"], rtol=1e-12, atol=1e-17)


def test_adam_matches_reference_bitwise():
    g = golden("adam.npz")
    names = ("a", "b", "c")
    p = {k: g["init_" + k].copy() for k in names}
    opt = oadam.AdamOracle(p, 3e-3)
    for t in range(3):
        opt.step({k: g[f"g{t}_{k}"] for k in names if f"g{t}_{k}" in g})
    for k in names:
        assert np.array_equal(p[k], g["final_" + k])


def test_mlp_matches_reference():
    g = golden("mlp.npz")
    p = omlp.init_params(47, seed=3)
    for k in omlp.NAMES:
        assert np.array_equal(p[k], g["init_" + k]), k
    np.testing.assert_allclose(omlp.predict(p, g["X"]), g["pred"], rtol=1e-12, atol=1e-14)
    for loss in ("rmse", "ranking"):
        l, gr = omlp.loss_and_gradients(p, g["X"][:16], g["y"][:16], loss)
        assert l == pytest.approx(float(g[f"{loss}_loss"]), rel=1e-12)
        for k in omlp.NAMES:
            np.testing.assert_allclose(gr[k], g[f"{loss}_g_{k}"], rtol=1e-10, atol=1e-14)
    for loss in ("rmse", "ranking"):
        pf, curve = omlp.fit(g["fit_X"], g["fit_y"], batch_size=8, epochs=3, lr=3e-3, loss=loss,
                             seed=1, eval_set=(g["fit_Xv"], g["fit_yv"]))
        for k in omlp.NAMES:
            np.testing.assert_allclose(pf[k], g[f"fit_{loss}_{k}"], rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(np.array(curve), g[f"fit_{loss}_curve"], rtol=1e-10)


def test_tuner_small_matches_reference():
    g = golden("tuner.npz")
    seqs = unpack_seqs(g["small_steps"], g["small_off"], g["small_ctx"])
    p = otuner.init_params(1, layers=2, hidden=4)
    for k, v in p.items():
        assert np.array_equal(v, g["small_init_" + k]), k
    np.testing.assert_allclose(otuner.predict(p, seqs), g["small_pred"], rtol=1e-12)
    for loss in ("rmse", "ranking"):
        l, gr = otuner.loss_and_gradients(p, seqs, g["small_y"], loss)
        assert l == pytest.approx(float(g[f"small_{loss}_loss"]), rel=1e-12)
        for k in p:
            np.testing.assert_allclose(gr[k], g[f"small_{loss}_g_{k}"], rtol=1e-9, atol=1e-14)


def test_tuner_default_matches_reference():
    g = golden("tuner.npz")
    seqs = unpack_seqs(g["dflt_steps"], g["dflt_off"], g["dflt_ctx"])
    p = otuner.init_params(0)
    names = list(p)
    np.testing.assert_array_equal([p[k].sum() for k in names], g["dflt_init_sum"])
    np.testing.assert_array_equal([np.abs(p[k]).sum() for k in names], g["dflt_init_abs"])
    np.testing.assert_allclose(otuner.predict(p, seqs), g["dflt_pred"], rtol=1e-12)
    np.testing.assert_allclose(otuner.predict(p, seqs, chunk=7), g["dflt_pred_chunk7"], rtol=1e-12)
    for loss in ("rmse", "ranking"):
        l, gr = otuner.loss_and_gradients(p, seqs[:16], g["dflt_y"][:16], loss)
        assert l == pytest.approx(float(g[f"dflt_{loss}_loss"]), rel=1e-12)
        np.testing.assert_allclose([np.linalg.norm(gr[k]) for k in names],
                                   g[f"dflt_{loss}_gnorm"], rtol=1e-9)
        for k in ("head_W2", "head_b2", "attn_bq", "attn_bo", "lstm2_bw_b", "lstm0_fw_Wx"):
            np.testing.assert_allclose(gr[k], g[f"dflt_{loss}_g_{k}"], rtol=1e-8, atol=1e-15)


def test_tuner_training_trajectory_matches_reference():
    g = golden("tuner.npz")
    seqs = unpack_seqs(g["fit_steps"], g["fit_off"], g["fit_ctx"])
    y, grp = g["fit_y"], list(g["fit_groups"])
    for loss in ("rmse", "ranking"):
        p = otuner.init_params(9, layers=1, hidden=4)
        curve = otuner.train(p, seqs, y, epochs=2, lr=3e-3, batch_size=4, seed=9, loss=loss,
                             eval_set=(seqs, y), eval_groups=grp)
        for k in p:
            np.testing.assert_allclose(p[k], g[f"fit_{loss}_{k}"], rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(np.array(curve, dtype=np.float64), g[f"fit_{loss}_curve"],
                                   rtol=1e-9)
        head = set(otuner.groups(p)["head"])
        before = {k: v.copy() for k, v in p.items()}
        curve = otuner.train(p, seqs, y, epochs=2, lr=1e-3, batch_size=4, seed=9, seed_offset=9001,
                             trainable=head, loss=loss)
        for k in p:
            np.testing.assert_allclose(p[k], g[f"cont_{loss}_{k}"], rtol=1e-9, atol=1e-13)
            if k not in head:
                assert np.array_equal(p[k], before[k])


def test_filter_stats_match_reference():
    g = golden("sampling.npz")
    for ci, (q, mr) in enumerate(g["cases"]):
        thr, keep, surv, tkeep = osamp.filter_stats(g["flops"], g["cost"], g["valid"],
                                                    g["offsets"], q, int(mr))
        np.testing.assert_array_equal(thr, g[f"thr_{ci}"])
        np.testing.assert_array_equal(keep, g[f"keep_{ci}"])
        np.testing.assert_array_equal(tkeep, g[f"tkeep_{ci}"])
    for qi, q in enumerate(g["tie_q"]):
        thr, *_ = osamp.filter_stats(g["tie_flops"], g["tie_cost"], g["tie_valid"], g["tie_off"],
                                     q, 1)
        np.testing.assert_array_equal(thr, g[f"tie_thr_{qi}"])
    raw = osamp.raw_task_weights(g["task_flops"], list(g["task_ops"]))
    tot = sum(raw)
    np.testing.assert_array_equal([w / tot for w in raw], g["weights"])


def test_gbdt_oracle_matches_reference_trees_bitwise():
    """oracle/gbdt.py (level-wise growth + DFS renumbering, the GPU's
    construction) reproduces the reference's trees, curves and predictions
    bit for bit on every golden case."""
    from oracle import gbdt as ogbdt

    g = golden("gbdt.npz")
    for name in g["names"]:
        nt, md, lr, ml = g[f"{name}_params"]
        base, trees, curve = ogbdt.fit(g[f"{name}_X"], g[f"{name}_y"], num_trees=int(nt), max_depth=int(md),
                                       learning_rate=float(lr), min_samples_leaf=int(ml),
                                       eval_set=(g[f"{name}_Xv"], g[f"{name}_yv"]))
        assert base == g[f"{name}_w_base"][0]
        assert np.array_equal([t[0].shape[0] for t in trees], g[f"{name}_w_node_counts"]), name
        for i, key in enumerate(("feature", "threshold", "left", "right", "value")):
            assert np.array_equal(np.concatenate([t[i] for t in trees]), g[f"{name}_w_{key}"]), (name, key)
        assert np.array_equal(np.array(curve, dtype=np.float64), g[f"{name}_curve"]), name
        assert np.array_equal(ogbdt.predict(base, trees, float(lr), g[f"{name}_Xv"]), g[f"{name}_pred"]), name
