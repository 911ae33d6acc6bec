#!/bin/bash
# Bench + evidence for one tag: default bench line, reference arm, launch list,
# and `ncu --set full` of one FULL-SIZE training epoch (the bench's own launch).
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py > $OUT/${TAG}_bench.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/${TAG}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tuner_train -s 3 -c 1 \
    -o $OUT/${TAG}_prof_train_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > $OUT/${TAG}_prof_train_full.log 2>&1
ls -la $OUT | tail -20
