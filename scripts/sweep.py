"""Throughput sweep over the BASELINE workloads: every config in its primary mode
and K values, against the dense per-timestep baseline through the same kernels
(the paper's comparison, Tables tab:speedup / tab:dvsg), plus the spike-density
independence check of SURVEY.md section 8(d).

    python scripts/sweep.py [--out gpurun_out/sweep.jsonl] [--iters 5] [--only C5]

One JSON line per (config, mode, K): device ms per forward of the whole conv stack
(CUDA events on the launch stream, inputs resident, after warm-up), input
spike-frames/s, per-layer ms and engines, logical conv calls per sample
(sum_l T_l / K_l) and the speedup over the config's dense run,
the slowest layer's roofline fractions (LIF ops vs the 148 x 128-lane ALU issue peak,
useful conv FLOP/s vs the tensor peak of its operand type, packed bytes vs HBM) and the
SM clocks / throttle reasons sampled while the line was timed.  "+FC" lines are the
whole networks (conv stack + FC head, the DVS one with the VotingLayer readout).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2603_13810_b200 import configs, network, tacsnn  # noqa: E402
import bench  # noqa: E402  (peaks, clock sampler, per-layer work counts)

PEAKS = bench.load_peaks()


def roofline(specs, layer_ms, B, engines):
    """Roofline fractions of the slowest layer (per-sample work x B / its time)."""
    i = max(range(len(layer_ms)), key=lambda j: layer_ms[j])
    t = layer_ms[i] / 1e3
    ns = bench.neuron_steps_per_sample(specs)[i] * B
    fl = bench.useful_flops_per_sample(specs)[i] * B
    by = bench.algorithmic_bytes_per_sample(specs)[i] * B
    alu_peak = 148 * 128 * PEAKS["sm_max_mhz"] * 1e6
    s = specs[i]
    int8 = engines[i] == "tcgen05" and s.C_in % 32 == 0 and s.H > 1
    tc_peak = PEAKS["bf16"] * 1e12 * (2.0 if int8 else 1.0)
    return {"layer": i, "ms": layer_ms[i], "alu_frac": bench.LIF_ALG_OPS * ns / t / alu_peak,
            "tensor_frac": fl / t / tc_peak, "tensor_peak": "int8 (2 x measured bf16)" if int8 else "bf16 (measured)",
            "hbm_frac": by / t / (PEAKS["hbm"] * 1e9)}

RUNS = [
    ("C1", "dense", 1), ("C1", "tac", 4), ("C1", "tactp", 4),
    ("C2", "dense", 1), ("C2", "tac", 2), ("C2", "tac", 4), ("C2", "tac", 8),
    ("C3", "dense", 1), ("C3", "tac", 8),
    ("C4", "dense", 1), ("C4", "tactp", 2), ("C4", "tac", 2),
    ("C5", "dense", 1), ("C5", "tactp", 2), ("C5", "tactp", 4), ("C5", "tactp", 8), ("C5", "tac", 4),
]
# the paper's MNIST setting T = 25 with K = 4 / 8 / 16: partial last groups
RUNS_T25 = [("C2", "dense", 1), ("C2", "tac", 4), ("C2", "tac", 8), ("C2", "tac", 16)]


def time_forward(net, x, iters):
    stream = torch.cuda.current_stream()
    for _ in range(2):
        net.forward(x)
    torch.cuda.synchronize()
    nL = len(net.specs)
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(nL)] for _ in range(iters)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(iters):
        y = x
        for li, (spec, prep) in enumerate(zip(net.specs, net.prepared)):
            evs[i][li][0].record(stream)
            y = network.flatten_for(spec, y)   # FC head: the previous map as one packed row
            y, _, _ = tacsnn.conv_lif(spec, prep, y, want_counts=(li == nL - 1))  # readout: last layer
            evs[i][li][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / iters
    layer_ms = [sum(evs[i][li][0].elapsed_time(evs[i][li][1]) for i in range(iters)) / iters
                for li in range(nL)]
    return ms, layer_ms


def time_graph(net, x, iters):
    """Same forward replayed from a CUDA graph (Network.capture)."""
    graph, _ = net.capture(x)
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(iters):
        graph.replay()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / iters


def density_check(iters, out):
    """Same layer (C4 layer 1: 128->128 @64x64, TAC-TP K=2), inputs of density
    0.01 vs 0.5: the conv is a dense contraction, so the time must not depend on
    the spike density (the paper's own premise)."""
    cfg = configs.CONFIGS["C4"]
    spec = configs.layer_plan(cfg, B=64)[1]
    w, b = configs.layer_weights(cfg)[1]
    net = network.Network([spec], [(w, b)])
    res = {}
    g = torch.Generator(device="cuda").manual_seed(0)
    for rho in (0.01, 0.5):
        x = tacsnn.pack((torch.rand((spec.T, spec.B, spec.C_in, spec.H, spec.W), device="cuda",
                                    generator=g) < rho).to(torch.uint8))
        ms, _ = time_forward(net, x, iters)
        res[str(rho)] = ms
    line = {"check": "density_independence", "layer": "C4 L1 128->128 @64x64 TAC-TP K=2, B=64",
            "ms_rho_0.01": res["0.01"], "ms_rho_0.5": res["0.5"],
            "ratio": res["0.5"] / res["0.01"]}
    print(json.dumps(line), flush=True)
    out.write(json.dumps(line) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    dense_ms = {}
    with open(a.out, "w") as out:
        for name, mode, K in RUNS:
            if a.only and name != a.only:
                continue
            cfg = configs.CONFIGS[name]
            specs = configs.layer_plan(cfg, mode=mode, K=K)
            net = network.Network(specs, configs.layer_weights(cfg))
            x = tacsnn.pack(configs.make_inputs(cfg, device="cuda"))
            clk = bench.ClockSampler(0)
            clk.start()
            ms, layer_ms = time_forward(net, x, a.iters)
            graph_ms = time_graph(net, x, max(a.iters, 20)) if name in ("C1", "C2", "C3", "C4") else None
            clocks = clk.stop()
            frames = cfg.B * cfg.T
            if mode == "dense":
                dense_ms[name] = ms
            line = {"config": name, "mode": mode, "K": K, "B": cfg.B, "T": cfg.T,
                    "ms_per_forward": ms, "frames_per_s": frames / (ms / 1e3),
                    "speedup_vs_dense": (dense_ms[name] / ms) if name in dense_ms else None,
                    "conv_calls_per_sample": configs.conv_calls(cfg, mode, K),
                    "layer_ms": layer_ms, "engines": net.engines(),
                    "graph_ms_per_forward": graph_ms,
                    "graph_frames_per_s": None if graph_ms is None else frames / (graph_ms / 1e3),
                    "roofline": roofline(specs, layer_ms, cfg.B, net.engines()), "clocks": clocks}
            print(json.dumps(line), flush=True)
            out.write(json.dumps(line) + "\n")
            del net, x
            torch.cuda.empty_cache()
        if not a.only:
            t25_dense = None
            for name, mode, K in RUNS_T25:
                cfg = configs.CONFIGS[name]
                specs = configs.layer_plan(cfg, mode=mode, K=K, T=25)
                net = network.Network(specs, configs.layer_weights(cfg))
                x = tacsnn.pack(configs.make_inputs(cfg, T=25, device="cuda"))
                ms, layer_ms = time_forward(net, x, a.iters)
                g_ms = time_graph(net, x, max(a.iters, 20))
                if mode == "dense":
                    t25_dense = g_ms
                line = {"config": name + "@T25", "mode": mode, "K": K, "B": cfg.B, "T": 25,
                        "ms_per_forward": ms, "graph_ms_per_forward": g_ms,
                        "frames_per_s": cfg.B * 25 / (ms / 1e3),
                        "graph_speedup_vs_dense": t25_dense / g_ms,
                        "conv_calls_per_sample": configs.conv_calls(cfg, mode, K, T=25),
                        "layer_ms": layer_ms, "engines": net.engines(),
                        "partial": [s.partial for s in specs]}
                print(json.dumps(line), flush=True)
                out.write(json.dumps(line) + "\n")
            # the whole networks (conv stack + FC head): MNIST / FMNIST with
            # the spike-count readout, DVS with the VotingLayer (tac_vote on the last counts)
            for name, runs in (("C2", (("dense", 1), ("tac", 4), ("tac", 8))), ("C3", (("dense", 1), ("tac", 8))),
                               ("C4", (("dense", 1), ("tactp", 2), ("tac", 2))),
                               ("C5", (("dense", 1), ("tactp", 4)))):
                cfg = configs.CONFIGS[name]
                d_ms = None
                for mode, K in runs:
                    specs = configs.network_plan(cfg, mode=mode, K=K)
                    net = network.Network(specs, configs.network_weights(cfg),
                                          voters=configs.VOTERS[configs.head_kind(cfg)])
                    x = tacsnn.pack(configs.make_inputs(cfg, device="cuda"))
                    clk = bench.ClockSampler(0)
                    clk.start()
                    ms, layer_ms = time_forward(net, x, a.iters)
                    g_ms = time_graph(net, x, max(a.iters, 20)) if name != "C5" else ms
                    clocks = clk.stop()
                    d_ms = g_ms if mode == "dense" else d_ms
                    nconv = len(cfg.layers)
                    line = {"config": name + "+FC", "mode": mode, "K": K, "B": cfg.B, "T": cfg.T,
                            "ms_per_forward": g_ms, "eager_ms_per_forward": ms,
                            "graph_ms_per_forward": g_ms if name != "C5" else None,
                            "frames_per_s": cfg.B * cfg.T / (g_ms / 1e3), "speedup_vs_dense": d_ms / g_ms,
                            "conv_calls_per_sample": sum(-(-s.T // s.K) for s in specs),
                            "layer_ms": layer_ms, "fc_ms": sum(layer_ms[nconv:]),
                            "fc_share": sum(layer_ms[nconv:]) / sum(layer_ms),
                            "engines": net.engines(), "clocks": clocks}
                    print(json.dumps(line), flush=True)
                    out.write(json.dumps(line) + "\n")
                    del net, x
                    torch.cuda.empty_cache()
            density_check(a.iters, out)


if __name__ == "__main__":
    main()
