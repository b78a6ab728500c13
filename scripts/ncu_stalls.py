"""Stall-sample breakdown of an ncu report by execution-count class (read here, no GPU).

    python scripts/ncu_stalls.py gpurun_out/l0.ncu-rep [--top 30]
Instructions are grouped by how often they executed (role loops of the fused kernel
execute a characteristic number of times); for each class the stall reasons summed
over its instructions are printed, then the most-sampled instructions.
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    body = rows[2:]
    isrc, iex, ism = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    reasons = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    cls = collections.defaultdict(lambda: [0, 0, collections.Counter(), 0])
    for r in body:
        n = int(r[iex] or 0)
        s = int(r[ism] or 0)
        c = cls[n]
        c[0] += 1
        c[1] += s
        c[3] += n
        for i, name in reasons:
            v = int(r[i] or 0)
            if v:
                c[2][name[6:]] += v
    tot = sum(c[1] for c in cls.values())
    print(f"total stall samples {tot}")
    for n, (ni, s, rc, ex) in sorted(cls.items(), key=lambda kv: -kv[1][1])[:8]:
        print(f"exec count {n:>10d}: {ni:5d} instrs, {ex / 1e6:8.1f} M warp-instr, samples {s:8d} "
              f"({100 * s / max(tot, 1):5.1f}%)  " + ", ".join(f"{k} {v}" for k, v in rc.most_common(6)))
    print("top sampled instructions:")
    srt = sorted(body, key=lambda r: -int(r[ism] or 0))[:top]
    for r in srt:
        rc = sorted(((int(r[i] or 0), name[6:]) for i, name in reasons), reverse=True)[:3]
        print(f"  {r[0][-6:]} n={int(r[iex] or 0):>9d} s={int(r[ism] or 0):>6d} {r[isrc].strip()[:60]:60s} "
              + " ".join(f"{nm}:{v}" for v, nm in rc if v))


if __name__ == "__main__":
    main()
