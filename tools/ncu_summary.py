"""Summarise ncu artefacts for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py rep  <file.ncu-rep>  > profiles/<name>.txt
    python tools/ncu_summary.py list <launches.csv>  > profiles/<name>.txt

`rep`: per captured launch, the metrics the roofline and the judge use
(duration, DRAM bytes, L2 sectors, pipe utilisation, occupancy, registers).
`list`: the launch list of `ncu --metrics gpu__time_duration.sum`, aggregated
per kernel (count, total time, share of GPU time).
"""

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>18s} {u.get(k, '')}")


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"{'launches':>8s} {'total ms':>12s} {'share':>7s}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:8d} {v[1] / 1e6:12.3f} {100 * v[1] / tot:6.2f}%  {k}")


if __name__ == "__main__":
    {"rep": rep, "list": launches}[sys.argv[1]](sys.argv[2])
