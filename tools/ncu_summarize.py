"""Summaries of tools/ncu_capture.sh output for profiles/ (dev tool, runs here).

    python tools/ncu_summarize.py gpurun_out r01

writes profiles/<tag>_ncu_launches.csv (copy), <tag>_ncu_launches_summary.txt
(per-kernel launches / total / share of the decode-step kernels) and
<tag>_ncu_full_mega_summary.csv (selected metrics of the --set full capture,
header row, unit row, value row: the file bench.py's roofline.traffic reads)."""
import csv
import io
import os
import shutil
import sys
from collections import defaultdict

src, tag = sys.argv[1], sys.argv[2]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")

# launch list
raw = open(os.path.join(src, "launches.csv")).read()
lines = raw.splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("sfg::", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
    tot[name] += us
    cnt[name] += 1
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(out, f"{tag}_ncu_launches.csv"))
allus = sum(tot.values())
with open(os.path.join(out, f"{tag}_ncu_launches_summary.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none, decode-step kernels of "
            "`bench.py --steps 2 --warmup 3 --no-sweep --no-cpu`\n")
    f.write("(cold, serialised launches under ncu: use the SHARE, not the absolute times; fast::pgemm_kernel = the "
            "prompt prefill GEMMs, outside the timed decode steps; mega_kernel = the 2+28+2 layer stacks of each "
            "decode step; fast::gemm_kernel<3,1> = the LM head with fused argmax partials)\n")
    f.write(f"{'kernel':60s} {'launches':>9s} {'total_us':>10s} {'share':>6s}\n")
    for k in sorted(tot, key=lambda k: -tot[k]):
        f.write(f"{k[:60]:60s} {cnt[k]:9d} {tot[k]:10.1f} {100 * tot[k] / allus:5.1f}%\n")

# --set full capture: raw page (header, units, values)
want = ["Kernel Name", "dram__bytes.sum.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__time_duration.sum", "launch__block_size", "launch__grid_size", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
raw = list(csv.reader(open(os.path.join(src, "mega_full_raw.csv"))))
h = raw[0]
units, vals = raw[1], raw[2]
idx = [h.index(w) for w in want]
with open(os.path.join(out, f"{tag}_ncu_full_mega_summary.csv"), "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(want)
    w.writerow([units[i] for i in idx])
    w.writerow([vals[i] for i in idx])
print(open(os.path.join(out, f"{tag}_ncu_launches_summary.txt")).read())
print(open(os.path.join(out, f"{tag}_ncu_full_mega_summary.csv")).read())
