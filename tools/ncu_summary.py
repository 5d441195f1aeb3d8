"""Summarise an .ncu-rep: per kernel duration, DRAM bytes, throughputs,
occupancy, stall reasons and the instruction mix (SASS opcode histogram)."""
import csv
import io
import subprocess
import sys
from collections import Counter

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
]


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True).stdout


def main(path, sass=False):
    rows = list(csv.reader(io.StringIO(ncu([path, "--page", "raw", "--csv"]))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in data:
        name = r[ix["Kernel Name"]][:90]
        print(f"== {name}")
        for m in METRICS:
            if m in ix:
                print(f"   {m} = {r[ix[m]]} {units[ix[m]]}")
        st = []
        for h, i in ix.items():
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.1:
                    st.append((v, h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)))
    if sass:
        for k in range(len(data)):
            out = ncu([path, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(k), "--launch-count", "1"])
            rows = list(csv.reader(io.StringIO(out)))
            hdr = rows[1]
            ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
            c, tot = Counter(), 0
            for r in rows[2:]:
                if len(r) > ie and r[ie].isdigit():
                    n = int(r[ie])
                    toks = r[src].split()
                    if not toks:
                        continue
                    op = toks[1] if toks[0].startswith("@") else toks[0]
                    c[op.split(".")[0]] += n
                    tot += n
            print(f"   [{k}] inst mix (warp-level, total {tot}):", ", ".join(f"{o}={v / tot * 100:.1f}%" for o, v in c.most_common(14)))


if __name__ == "__main__":
    main(sys.argv[1], sass="--sass" in sys.argv)
