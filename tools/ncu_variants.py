"""Table of the ncu --set full captures of the three variants of the same
kernel (tools/gpu_ncu_variants.sh): time, DRAM GB/s vs the copy peak, tensor
pipe utilisation, useful vs issued FLOPs. Writes profiles/<tag>_ncu_variants.md."""
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11608_b200 import _core  # noqa: E402

N = 2048
USEFUL = 2 * N * 112 * 112 * 64 * 7 * 7 * 3  # R50 conv1, count_macs x 2
def _peaks():
    """MEASURED_PEAKS.json (driver-written), else the B200_PROFILING.md fallback, labelled."""
    import json
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


PEAK_GBS, PEAK_TF, PEAK_SRC = _peaks()
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def scale(v, unit):
    v = float(v.replace(",", ""))
    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
                "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}.get(unit, 1)


def main(tag):
    plans = {
        "fold": _core.FoldedConv([N, 224, 224, 3], [7, 7, 3, 64], 2, 2, 3, 3, "bf16", 0, 0, "fold").device,
        "zeropad": _core.FoldedConv([N, 224, 224, 8], [7, 7, 8, 64], 2, 2, 3, 3, "bf16", 0, 0, "fold").device,
        "unfolded": _core.FoldedConv([N, 224, 224, 3], [7, 7, 3, 64], 2, 2, 3, 3, "bf16", 0, 0, "unfolded").device,
    }
    lines = ["# R50 conv1, n=2048, bf16: three variants of the same tcgen05 kernel (ncu --set full, one launch)", "",
             "ncu times are cold-cache, serialised, one launch under the profiler (clock-control none).", "",
             f"Peaks: HBM {PEAK_GBS:.1f} GB/s, bf16 {PEAK_TF:.1f} TF/s ({PEAK_SRC}).", "",
             f"| variant | time ms | DRAM read+write GB | DRAM GB/s (frac of {PEAK_GBS:.0f}) | tensor pipe % | TC smem wavefronts % | useful TFLOP/s (frac of {PEAK_TF:.0f}) | issued TFLOP/s | useful/issued | instructions |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for v in ("fold", "zeropad", "unfolded"):
        rep = os.path.join(ROOT, "gpurun_out", f"prof_var_{v}.ncu-rep")
        if not os.path.exists(rep):
            continue
        val, unit = raw(rep)
        t = scale(val["gpu__time_duration.sum"], unit["gpu__time_duration.sum"])
        by = scale(val["dram__bytes_read.sum"], unit["dram__bytes_read.sum"]) + \
            scale(val["dram__bytes_write.sum"], unit["dram__bytes_write.sum"])
        issued = 2 * plans[v]["issued_macs"]
        tp = val.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "n/a")
        tcw = val.get("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "n/a")
        lines.append(f"| {v} | {t * 1e3:.3f} | {by / 1e9:.2f} | {by / t / 1e9:.0f} ({by / t / 1e9 / PEAK_GBS:.2f}) | {tp} | "
                     f"{tcw} | {USEFUL / t / 1e12:.0f} ({USEFUL / t / 1e12 / PEAK_TF:.3f}) | {issued / t / 1e12:.0f} | {USEFUL / issued:.3f} | "
                     f"{val.get('smsp__inst_executed.sum', 'n/a')} |")
    out = os.path.join(ROOT, "profiles", f"{tag}_ncu_variants.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1g")
