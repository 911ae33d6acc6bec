#!/bin/bash
# compute-sanitizer over every hot kernel (tools/sanitize_workload.py):
# memcheck for all parts, racecheck / synccheck (shared-memory hazards,
# barrier misuse) per part.  Logs -> gpurun_out/sanitize_*.log
#   gpurun --timeout 3000 -- 'bash tools/sanitize.sh'
OUT=gpurun_out
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for part in train train_multiround dp predict mlp metrics gbdt; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_workload.py $part > $OUT/sanitize_${tool}_${part}.log 2>&1
    echo "$tool $part rc=$?" | tee -a $OUT/sanitize_summary.txt
  done
done
