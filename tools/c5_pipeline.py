"""North-star config 5 end to end through the reference's own workflow code
(transfer.py:107-278, sampling.py:128-200, models.py), with the B200 kernels
installed (or, with --cpu, the unmodified reference on the host):

  source pretrain on the pruned source dataset
      prune_dataset(source, SamplerConfig(target_fraction=0.55))  (K2 statistics)
      train_tuner(pruned source, within_task split)              (fused training)
  adapt_hardware(model, cpu-xeon24 -> gpu-t4ish)
  fine_tune on a 40 % budget of the destination's train records
      heads-only (frozen-stack cache kernel) and full scope
  evaluate on the destination's test split                       (K1 + K10)

Prints one JSON line: wall seconds per stage and the quality numbers.

    python tools/c5_pipeline.py [--kernels 10] [--records 96] [--epochs 200] [--cpu]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", type=int, default=10)
    ap.add_argument("--records", type=int, default=96)
    ap.add_argument("--epochs", type=int, default=200)
    ap.add_argument("--ft-epochs", type=int, default=300)
    ap.add_argument("--cpu", action="store_true", help="the unmodified reference (no install())")
    args = ap.parse_args()

    import tensortune.cli  # noqa: F401
    import tensortune.models as tm
    import tensortune.sampling as ts
    import tensortune.transfer as tt
    from tensortune.benchmarks import transfer_benchmark
    from tensortune.data import Dataset
    from tensortune.hardware import registry_by_id
    from tensortune.splits import split

    if not args.cpu:
        from paper_2304_05430_b200.install import install

        install()
    out = {"impl": "reference-cpu" if args.cpu else "b200", "kernels": args.kernels,
           "records_per_task": args.records, "epochs": args.epochs, "ft_epochs": args.ft_epochs}
    wall = {}

    def timed(name, fn):
        t0 = time.perf_counter()
        r = fn()
        wall[name] = round(time.perf_counter() - t0, 3)
        return r

    _, src_ds, dst_ds = timed("generate", lambda: transfer_benchmark(seed=0, n_kernels=args.kernels,
                                                                     records_per_task=args.records))
    by_id = registry_by_id()
    cpu, gpu = by_id["cpu-xeon24"], by_id["gpu-t4ish"]
    pruned, prep = timed("prune_0.55", lambda: ts.prune_dataset(src_ds, ts.SamplerConfig(target_fraction=0.55,
                                                                                      seed=0)))
    out["prune_records"] = [len(src_ds.records), len(pruned.records)]
    pre, pre_rep = timed("pretrain", lambda: tm.train_tuner(pruned, split(pruned, "within_task", 0.25, 0),
                                                            tm.TrainConfig(epochs=args.epochs, seed=0)))
    out["pretrain_val_rmse"] = pre_rep.val_rmse
    dsplit = split(dst_ds, "within_task", 0.25, 0)
    train_records = [r for r in dst_ds.records if r.record_id in dsplit.train_ids]
    dst_train = Dataset.build(list(dst_ds.hardware), list(dst_ds.tasks), train_records)
    budget = int(0.4 * len(train_records))
    adapted, mapping = timed("adapt", lambda: tt.adapt_hardware(pre, cpu, gpu))
    for scope in ("heads-only", "full"):
        cfg = tt.TransferConfig(target=gpu.target_id, record_budget=budget, fine_tune_scope=scope,
                                fine_tune_epochs=args.ft_epochs, learning_rate=1e-3, seed=0)
        tuned, rep = timed(f"fine_tune_{scope}", lambda cfg=cfg: tt.fine_tune(adapted, dst_train, cfg, mapping))
        ev = timed(f"evaluate_{scope}", lambda tuned=tuned: tm.evaluate(tuned, dst_ds, dsplit))
        out[f"{scope}_holdout_pca_before_after"] = [rep.pca_before, rep.pca_after]
        out[f"{scope}_test_pca"] = ev.test_pairwise_accuracy
    out["budget_records"] = budget
    out["wall_s"] = wall
    out["wall_total_s"] = round(sum(wall.values()), 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
