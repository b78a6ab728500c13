"""Instruction-count classes of an ncu report (read here, no GPU).

    python scripts/ncu_classes.py gpurun_out/c5l0.ncu-rep [--dump N]
Groups SASS instructions by execution count (each role loop of the fused kernel runs a
characteristic number of times: per tile, per group, per warp) and prints, per class,
the instruction count, the warp-instructions executed, the stall samples and the opcode
mix; --dump N prints the instructions of the class executed N times.
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    dump = int(sys.argv[sys.argv.index("--dump") + 1]) if "--dump" in sys.argv else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, body = rows[1], rows[2:]
    isrc, iex = h.index("Source"), h.index("Instructions Executed")
    ism = h.index("Warp Stall Sampling (All Samples)")
    cls = collections.defaultdict(lambda: [0, 0, 0, collections.Counter()])
    for r in body:
        n = int(r[iex] or 0)
        if n == 0:
            continue
        c = cls[n]
        c[0] += 1
        c[1] += n
        c[2] += int(r[ism] or 0)
        op = r[isrc].split()
        o = op[1] if op[0].startswith("@") else op[0]
        c[3][o.split(".")[0]] += 1
        if dump == n:
            print(f"{r[0][-6:]} {r[isrc].strip()[:90]:90s} {r[ism]}")
    tot = sum(c[1] for c in cls.values())
    print(f"total warp-instructions {tot / 1e6:.1f} M")
    for n, (ni, ex, sm, ops) in sorted(cls.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"exec {n:>10d}: {ni:4d} instrs {ex / 1e6:9.1f} M ({100 * ex / tot:5.1f}%) samples {sm:7d}  "
              + " ".join(f"{k}:{v}" for k, v in ops.most_common(8)))


if __name__ == "__main__":
    main()
