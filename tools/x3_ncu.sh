# ncu evidence for the fp32 tensor-core tuner scorer (tools/x3_probe.py --quick):
# launch list + one --set full capture of each kernel, summaries in gpurun_out/
TAG=${1:-x3}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'lstm_x3|attn_|x3_prepare' --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/x3_probe.py --quick > /dev/null 2>&1
python tools/ncu_summary.py list gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'lstm_x3|attn_' -c 2 \
  -o gpurun_out/${TAG}full python tools/x3_probe.py --quick > gpurun_out/${TAG}ncu.log 2>&1
python tools/ncu_summary.py rep gpurun_out/${TAG}full.ncu-rep > gpurun_out/${TAG}_full.txt 2>&1
