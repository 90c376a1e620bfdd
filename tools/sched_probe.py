"""Write the R50 (or given) M-tile schedule as a text table for tools/probes/sched_probe.cu."""
import sys
sys.path.insert(0, ".")
from paper_2601_11608_b200 import _abi as A  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sched_table.txt"
sc = A.schedule_describe(A.make_desc(8192, 224, 224, 3, 7, 7, 64, 2, 2, 3, 3), 0, 0, A.WF_BF16)
e = sc["entries"]
with open(out, "w") as f:
    for i in range(0, len(e), 7):
        a_off, lbo, b_off, meta, col = e[i:i + 5]
        n = ((meta >> 22) & 0x1FF) * 8
        f.write(f"{a_off} {lbo} {b_off} {n} {col} {meta >> 31}\n")
print(out, len(e) // 7, "entries, kpair", sc["kpair"])
