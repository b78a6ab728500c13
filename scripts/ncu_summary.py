"""Summarise an ncu report (read here, no GPU): key throughput metrics, stall
reasons, and the hottest SASS regions by executed instructions / stall samples.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--sass]
"""
import collections
import csv
import io
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
]


def main():
    rep = sys.argv[1]
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:                      # one row per profiled launch
        d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
        print("kernel:", d.get("Kernel Name", ("?",))[0][:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k][0]:>16s} {d[k][1]}")
        stalls = {k: float(v[0] or 0) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")}
        print("  stall reasons (warps per issue):")
        for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
            print(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {v:.3f}")
    if "--sass" in sys.argv:
        rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
        hdr = rows[1]
        ia, isrc, iaddr = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Address")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        recs = []
        for r in rows[2:]:
            try:
                recs.append((int(r[iaddr], 16), int(r[ia] or 0), int(r[isamp] or 0), r[isrc]))
            except (ValueError, IndexError):
                pass
        recs.sort()
        tot = sum(n for _, n, _, _ in recs) or 1
        stot = sum(s for _, _, s, _ in recs) or 1
        print(f"  executed instructions: {tot}")
        cnt = collections.Counter(n for _, n, _, _ in recs)
        print("  most common per-instruction execution counts (count x #instrs):")
        for n, c in cnt.most_common(8):
            print(f"    {n} x {c} = {100.0 * n * c / tot:.1f}%")
        print("  top stall-sampled instructions:")
        base = recs[0][0]
        for a, n, s, src in sorted(recs, key=lambda x: -x[2])[:20]:
            print(f"    +{a - base:06x} {n:>10d} {100.0 * s / stot:5.1f}%  {src[:80]}")


if __name__ == "__main__":
    main()
