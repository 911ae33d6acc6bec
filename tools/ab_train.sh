#!/bin/bash
# A/B of training-kernel variants: bench step time (device) + phase marks +
# the training parity tests, per library (TT_LIB).  Usage:
#   gpurun -- 'bash tools/ab_train.sh TAG lib1.so lib2.so ...'
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
for L in "$@"; do
  n=$(basename $L .so)
  for rep in 1 2; do
    TT_LIB=$PWD/$L timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-extra > $OUT/${TAG}_${n}_bench$rep.log 2>&1
  done
  TT_LIB=$PWD/$L timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-extra --phases > $OUT/${TAG}_${n}_phases.log 2>&1
  TT_LIB=$PWD/$L timeout 900 python -m pytest -q -x tests/test_gpu_train_paths.py tests/test_gpu_dp_fused.py tests/test_gpu_tuner.py > $OUT/${TAG}_${n}_tests.log 2>&1
  echo "$n tests rc=$?" >> $OUT/${TAG}_summary.txt
  python - "$OUT" "$TAG" "$n" >> $OUT/${TAG}_summary.txt <<'PY'
import json, sys, glob
out, tag, n = sys.argv[1:4]
for f in sorted(glob.glob(f"{out}/{tag}_{n}_bench*.log")):
    ls = [x for x in open(f) if x.startswith("{")]
    if ls:
        d = json.loads(ls[-1]); print(n, f[-10:], round(d["value"]), "samples/s", round(d["ms_per_step"] / 16.384, 2), "us/step")
PY
done
cat $OUT/${TAG}_summary.txt
