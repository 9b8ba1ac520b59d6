"""Summarise an ncu report: per kernel duration, DRAM bytes, pipe utilisation,
top stall reasons, and the SASS instructions with the most stall samples."""
import csv
import io
import subprocess
import sys
from collections import Counter


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum"]


def main(rep, source_regex=None):
    h, units, rows = raw(rep)
    ki = h.index("Kernel Name")
    for r in rows:
        vals = dict(zip(h, r))
        print("==", r[ki][:90])
        for k in KEYS:
            if k in vals:
                print(f"   {k:70s} {vals[k]:>16s} {units[h.index(k)]}")
        st = []
        for k, v in vals.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        print("   stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:6]))
    if source_regex:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{source_regex}",
                              "--print-source", "sass"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h = rows[1]
        si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        c = Counter()
        tot = 0
        for r in rows[2:]:
            try:
                v = int(r[wi])
            except (ValueError, IndexError):
                continue
            tot += v
            toks = r[si].split()
            op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
            c[op.split(".")[0]] += v
        print(f"== stall samples by opcode ({source_regex}), total {tot}")
        for k, v in c.most_common(10):
            print(f"   {v / max(tot, 1) * 100:6.2f}% {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
