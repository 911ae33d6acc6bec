#!/bin/bash
# One gpurun call: GPU parity tests (incl. the reference's own suite through
# install()), smoke, the default bench line and the reference arm; with
# NCU=1 also the ncu launch list of the bench and `ncu --set full` captures
# of the top kernels (one full training epoch = the bench's launch; the
# scoring kernels at the bench's sizes).
#   gpurun --timeout 3600 -- 'bash tools/gpu_round.sh [tag]'
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_smi.txt 2>&1
lscpu > $OUT/${TAG}_lscpu.txt 2>&1
TT_REFSUITE_LOGDIR=$OUT/${TAG}_refsuite timeout 2400 python -m pytest tests -m gpu -q -rfE > $OUT/${TAG}_pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_smoke.log
timeout 900 python bench.py > $OUT/${TAG}_bench.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_bench_ref.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_bench_ref.log
if [ "${NCU:-0}" = "1" ]; then
# .ncu-rep files stay on the box (/tmp): gpurun copies back <= 64 MiB, so only
# the text summaries (tools/ncu_summary.py) come home
REP=/tmp/ncu_${TAG}
mkdir -p $REP
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra --phases > $OUT/${TAG}_phases.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $OUT/${TAG}_launches.log 2>&1
python tools/ncu_summary.py list $OUT/${TAG}_launches.csv > $OUT/${TAG}_launches.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tuner_train -s 3 -c 1 \
    -o $REP/train_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-extra > $OUT/${TAG}_prof_train_full.log 2>&1
python tools/ncu_summary.py rep $REP/train_full.ncu-rep > $OUT/${TAG}_ncu_full_train.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'tuner_predict|lstm_x3|attn_rows|attn_warp|mlp_predict|pca_tile|rank_sort|gbdt_predict' -c 30 \
    -o $REP/scoring python tools/scoring_profile_driver.py > $OUT/${TAG}_prof_scoring.log 2>&1
python tools/ncu_summary.py rep $REP/scoring.ncu-rep > $OUT/${TAG}_ncu_full_scoring.txt 2>&1
ls -la $REP
fi
ls -la $OUT | tail -30
