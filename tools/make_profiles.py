"""Copy the judged evidence from gpurun_out/ (scratch) into profiles/ (tracked).

  python tools/make_profiles.py TAG

writes
  profiles/TAG_launches.txt        per-kernel share of the bench's launch list (ncu gpu__time_duration)
  profiles/TAG_launches.csv        the raw launch list
  profiles/TAG_ncu_<rep>.txt       key metrics + top stall sites of each .ncu-rep (tools/ncu_summary.py)
  profiles/ncu_traffic.json        dram read+write bytes per launch of the bench-sized kernel (bench.py reads it)
  profiles/TAG_bench.json          the bench lines (ours + reference arm)
"""
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def ncu_rows(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    return rows[hdr], rows[hdr + 1:]


def launches(tag):
    src = os.path.join(OUT, "launches.csv")
    if not os.path.exists(src):
        return
    shutil.copy(src, os.path.join(PROF, f"{tag}_launches.csv"))
    h, rows = ncu_rows(src)
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows:
        agg[r[ik]].append(float(r[iv]))
    tot = sum(sum(v) for v in agg.values())
    with open(os.path.join(PROF, f"{tag}_launches.txt"), "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none -c 40 python bench.py --steps 4 --warmup 3 "
                "--no-e2e --no-cpu --no-verify\n(cold-cache, serialised: compare shares, not absolutes; the torch "
                "kernels are input synthesis and the zero-pad variant's setup, outside the timed region)\n\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{len(v):4d} launches {sum(v) / 1e3:10.1f} us {sum(v) / tot * 100:5.1f}%  "
                    f"mean {sum(v) / len(v) / 1e3:8.1f} us  {k[:110]}\n")


def reports(tag):
    for rep in sorted(glob.glob(os.path.join(OUT, "*.ncu-rep"))):
        name = os.path.splitext(os.path.basename(rep))[0]
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, "25"],
                             capture_output=True, text=True).stdout
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        extra = []
        if len(rows) > 2:
            want = ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
                    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
                    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                    "sm__cycles_elapsed.avg", "launch__registers_per_thread", "launch__grid_size",
                    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active")
            for k, u, v in zip(rows[0], rows[1], rows[2]):
                if k in want:
                    extra.append(f"{k:80s} {v:>18s} {u}")
        with open(os.path.join(PROF, f"{tag}_ncu_{name}.txt"), "w") as f:
            f.write(f"ncu --set full --clock-control none --import-source on -k regex:conv_fold ({name})\n\n")
            f.write("\n".join(extra) + "\n\n" + out)


def traffic():
    path = os.path.join(OUT, "traffic_r50_n8192.csv")
    if not os.path.exists(path):
        return
    h, rows = ncu_rows(path)
    vals = {r[h.index("Metric Name")]: float(r[h.index("Metric Value")]) for r in rows}
    tj = os.path.join(PROF, "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d["resnet50_conv1_b8192_224_nhwc_bf16_n8192"] = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    d["_how"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:conv_fold -c 1 "
                 "python tools/prof_conv.py r50 8192 (one launch of the bench-sized kernel)")
    json.dump(d, open(tj, "w"), indent=1)


def bench(tag):
    lines = []
    for name in ("bench.log", "bench_ref.log"):
        p = os.path.join(OUT, name)
        if os.path.exists(p):
            lines += [ln for ln in open(p).read().splitlines() if ln.startswith("{")]
    if lines:
        with open(os.path.join(PROF, f"{tag}_bench.jsonl"), "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    reports(tag)
    traffic()
    bench(tag)
    print(sorted(os.listdir(PROF)))
