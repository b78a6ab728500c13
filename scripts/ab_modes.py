"""A/B timing of variant builds on one C5 layer across modes (each variant in a
fresh process, round-robin twice): python scripts/ab_modes.py <layer> <B> lib_a.so lib_b.so"""
import os
import subprocess
import sys

L, B, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
for rep in (1, 2):
    for mode, K in (("dense", 1), ("tac", 4), ("tactp", 4)):
        for lib in libs:
            env = dict(os.environ, TACSNN_LIB=os.path.join("paper_2603_13810_b200", lib))
            out = subprocess.run([sys.executable, "scripts/profile_layer.py", "--config", "C5", "--layer", L,
                                  "--B", B, "--iters", "4", "--mode", mode, "--K", str(K)],
                                 env=env, capture_output=True, text=True, timeout=300).stdout
            t = [ln.split()[0] for ln in out.splitlines() if " ms " in ln][-2:]
            print(f"rep {rep} layer {L} {mode:6s} K{K} {lib:28s} {' '.join(t)}", flush=True)
