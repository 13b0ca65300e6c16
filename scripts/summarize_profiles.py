"""Turns a round's ncu artefacts (gpurun_out/<tag>_launches.csv from the
`--metrics gpu__time_duration.sum` pass over bench.py and gpurun_out/<tag>_full.ncu-rep from
the `--set full` pass over scripts/profile_step.py) into the tracked summaries under profiles/:

  profiles/<tag>_launches.csv      per-launch durations of the bench command (raw ncu CSV)
  profiles/<tag>_full_metrics.csv  selected --set full metrics per profiled kernel
  profiles/<tag>_traffic.json      DRAM bytes per launch per kernel (bench.py roofline.traffic)
  profiles/<tag>_kernels.md        the table the DESIGN.md roofline section cites

Usage: python scripts/summarize_profiles.py r1
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out")
DST = os.path.join(ROOT, "profiles")
os.makedirs(DST, exist_ok=True)

METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def short(name):
    return name.split("(")[0].replace("void ", "").replace("fc::", "")


def launches():
    src = os.path.join(SRC, f"{TAG}_launches.csv")
    shutil.copy(src, os.path.join(DST, f"{TAG}_launches.csv"))
    hdr, per = None, collections.OrderedDict()
    for r in csv.reader(open(src)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            per.setdefault(short(d["Kernel Name"]), []).append(float(d["Metric Value"].replace(",", "")) / 1e3)
    return per


def full():
    rep = os.path.join(SRC, f"{TAG}_full.ncu-rep")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    keep = [i for i, k in enumerate(hdr) if k == "Kernel Name" or k in METRICS]
    with open(os.path.join(DST, f"{TAG}_full_metrics.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow([hdr[i] for i in keep])
        w.writerow([units[i] for i in keep])
        res = []
        for r in rows[2:]:
            w.writerow([r[i] for i in keep])
            res.append({hdr[i]: r[i] for i in keep})
    return res


def main():
    per = launches()
    kern = full()

    def num(d, k):
        try:
            return float(d.get(k, "nan").replace(",", ""))
        except ValueError:
            return float("nan")

    traffic = {}
    for d in kern:
        rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")   # Mbyte
        traffic[short(d["Kernel Name"])] = (rd + wr) * 1e6
    json.dump({"note": "DRAM read+write bytes per launch from ncu --set full (cache flushed before each "
                       "profiled launch, so re-read operands that stay in L2 during a real step count here)",
               "bytes_per_launch": traffic}, open(os.path.join(DST, f"{TAG}_traffic.json"), "w"), indent=1)
    lines = [f"# {TAG}: ncu summaries of the B200 FastCLIP step (B = 5120, d = 512, fastclip_v3, 1 GPU)", "",
             "Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`python bench.py --steps 3 --warmup 3` (cold-cache, serialised launches; shares, not "
             "absolute step time). Full capture: `ncu --set full --clock-control none` over "
             "`scripts/profile_step.py`.", "",
             "| kernel | launches | mean us (launch list) | share | us (full) | SM GHz | DRAM MB r/w | tensor pipe % | SM thr % | L2 thr % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    tot = sum(sum(v) / len(v) for k, v in per.items() if not k.startswith("at::"))
    byk = {short(d["Kernel Name"]): d for d in kern}
    for k, v in per.items():
        if k.startswith("at::"):
            continue   # the bench's L2 flush (torch fill), not part of the step
        m = sum(v) / len(v)
        d = byk.get(k, {})
        lines.append(f"| {k} | {len(v)} | {m:.2f} | {100 * m / tot:.1f}% | {num(d, 'gpu__time_duration.sum'):.2f} | "
                     f"{num(d, 'sm__cycles_elapsed.avg.per_second'):.2f} | {num(d, 'dram__bytes_read.sum'):.1f} / "
                     f"{num(d, 'dram__bytes_write.sum'):.1f} | {num(d, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{num(d, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{num(d, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | {d.get('launch__registers_per_thread', '')} |")
    open(os.path.join(DST, f"{TAG}_kernels.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
