#!/usr/bin/env python
"""Benchmark of the Conv-LIF hot path (arXiv 2603.13810, TAC / TAC-TP / dense).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--mode tactp]
                    [--K 4] [--impl ours|reference] [--no-cpu-baseline]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU)

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself through
torch.distributed.run with N ranks (127.0.0.1); under torchrun WORLD_SIZE must equal
--gpus (a mismatch is an error, not a silent 1-rank run).

A step is one forward pass of the config's whole Conv-LIF stack (every row of
SURVEY.md section 8(a): aggregation, per-group conv, LIF, packed/pool/counts
outputs) over the rank's batch shard, followed by the NCCL all_gather of the
final-layer spikes and spike counts (the only collective, north_star).
Default workload: BASELINE config C5 (DVS128-shaped, 5 conv blocks, T=32, K=4,
batch 2048 sharded across the ranks, TAC-TP).  Metric: spike-frames/s at the
network input (B*T input frames per step), whole job.  Rank 0 prints ONE JSON
line.  `--impl reference` times the CPU oracle (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Conv-LIF spike-frames/s (dense/TAC/TAC-TP) at 1/8 B200; % tensor-pipe peak"
UNIT = "spike-frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--mode", default=None, help="dense | tac | tactp (default: config's)")
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--B", type=int, default=None, help="global batch (default: config's)")
    ap.add_argument("--engine", default="auto")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's global batch is sharded; weak: B per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-head", action="store_true", help="skip the whole-network (FC head) timing")
    ap.add_argument("--cpu-sample-T", type=int, default=8)
    ap.add_argument("--layer-detail", action="store_true")
    ap.add_argument("--no-v-final", action="store_true",
                    help="skip the extra timing with every layer writing v_final")
    ap.add_argument("--train", action="store_true",
                    help="time a training step (forward + surrogate-gradient BPTT backward) of the "
                         "config's network, TAC/TAC-TP against dense (SURVEY.md 8(f) #3)")
    ap.add_argument("--whole-net", action="store_true",
                    help="--train on the whole MNIST/FMNIST network (conv blocks + FC head)")
    ap.add_argument("--launcher-check", action="store_true",
                    help="CPU/gloo check of the rank launcher, shard and gather plumbing only "
                         "(no kernels, no timing; used by tests/test_bench_launcher.py)")
    return ap.parse_args()


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def ensure_ranks(a):
    """--gpus N: run as N ranks.  Outside torchrun, re-exec through torch.distributed.run;
    inside, insist that WORLD_SIZE == --gpus."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if a.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
                   "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
            os.execv(sys.executable, cmd)
        return
    if int(world) != a.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {a.gpus}; launch one rank per GPU")


# ------------------------------------------------------------------ helpers --
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"],
                    bf16_sustained=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    sm_max_mhz=d.get("sm_max_mhz", 1965.0), source="measured")
    # fallback stated in /opt/skills/guides/B200_PROFILING.md
    return dict(hbm=6650.0, bf16=1590.0, bf16_sustained=1400.0, sm_max_mhz=1965.0,
                source="fallback")


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def useful_flops_per_sample(specs):
    """Algorithmic conv FLOPs per sample of one forward: 2*Cout*H'W'*Cin*R*S per
    conv call, G = T/K calls per layer."""
    out = []
    for s in specs:
        hc, wc = s.conv_hw
        G = s.T // (1 if s.mode == "dense" else s.K)
        out.append(2.0 * s.C_out * hc * wc * s.C_in * s.R * s.S * G)
    return out


def neuron_steps_per_sample(specs):
    """LIF neuron-steps per sample of one forward: C_out * H' * W' * (LIF steps)."""
    out = []
    for s in specs:
        hc, wc = s.conv_hw
        steps = s.T // s.K if s.mode == "tac" else s.T
        out.append(float(s.C_out * hc * wc * steps))
    return out


LIF_ALG_OPS = 3.0  # per neuron-step: V <- beta V + Y (one FMA), threshold compare, reset subtract


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def algorithmic_bytes_per_sample(specs):
    """Packed spike bytes in + out per sample of one forward (no v_final)."""
    out = []
    for s in specs:
        T_out, Ho, Wo, wpr = s.out_shape()
        out.append(4.0 * (s.T * s.H * s.in_words_per_row + T_out * Ho * wpr) + 4.0 * s.C_out)
    return out


def dtype_note(specs, engines):
    """The arithmetic the step runs in, per operand path."""
    parts = []
    for i, (s, e) in enumerate(zip(specs, engines)):
        if e != "tcgen05":
            parts.append(f"L{i}: f32 (SIMT)")
        elif s.C_in % 32 == 0 and s.input == "spikes":
            parts.append(f"L{i}: u8 x 2 i8 slices -> s32")
        else:
            parts.append(f"L{i}: f16 x (f16 hi + lo) -> f32")
    return "; ".join(parts) + "; LIF f32"


def l2_note(specs, B):
    """Timing rule: inputs larger than L2, or a per-step working set that evicts them."""
    inb = 4.0 * specs[0].T * B * specs[0].H * specs[0].in_words_per_row
    ws = inb
    for s in specs:
        T_out, Ho, _, wpr = s.out_shape()
        ws += 4.0 * T_out * B * Ho * wpr
    return (f"per-rank packed input {inb / 2**20:.0f} MiB, per-step working set (input + every "
            f"layer's packed output) {ws / 2**20:.0f} MiB vs 126 MB L2: "
            + ("inputs alone exceed L2" if inb > 126e6 else
               "working set exceeds L2, so each step's input is evicted by the time it is re-read"
               if ws > 2 * 126e6 else "WARNING: working set fits L2"))


# --------------------------------------------------------------- CPU oracle --
def time_oracle(cfg, specs, weights, B, T_sample):
    """Run the oracle over the stack on a bounded sample; returns (seconds, frames)."""
    from oracle import oracle as O
    from paper_2603_13810_b200 import configs
    S = configs.make_inputs(cfg, B=B, T=T_sample).numpy()
    t0 = time.perf_counter()
    x = S
    t = T_sample
    for spec, (w, b) in zip(specs, weights):
        K = 1 if spec.mode == "dense" else min(spec.K, t)
        r = O.forward(x, w.numpy(), b.numpy(), K=K, mode=spec.mode, beta=spec.beta,
                      v_th=spec.v_th, reset=spec.reset, pad=spec.pad)
        x = O.or_pool2(r["out"]) if spec.out_pool == 2 else r["out"]
        if spec.mode == "tac":
            t //= K
    return time.perf_counter() - t0, B * T_sample


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(cfg, specs, weights, T_sample):
    from oracle import oracle as O
    thr = O.threads()
    B = max(1, min(thr, cfg.B))
    K = specs[0].K if specs[0].mode != "dense" else 1
    T_sample = max(K, (T_sample // K) * K)
    dt, frames = time_oracle(cfg, specs, weights, B, T_sample)
    # single-core figure: one sample through one thread
    O.set_threads(1)
    try:
        dt1, frames1 = time_oracle(cfg, specs, weights, 1, T_sample)
    finally:
        O.set_threads(thr)
    return {"value": frames / dt, "unit": UNIT, "cores": thr, "kind": "oracle",
            "single_core_value": frames1 / dt1, "cpu_model": cpu_model(),
            "sample": f"{cfg.name} stack, {B} samples x T={T_sample} (fp64 C oracle, OpenMP "
                      f"over samples), {dt:.1f} s; single core: 1 sample, {dt1:.1f} s"}


# --------------------------------------------------------------- reference --
def run_reference(a, cfg, specs_fn, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2603_13810_b200 import configs
    specs = specs_fn(1)
    weights = configs.layer_weights(cfg)
    thr = O.threads()
    B = max(1, min(thr, cfg.B))
    K = specs[0].K if specs[0].mode != "dense" else 1
    T_sample = K if specs[0].mode != "dense" else 1
    for _ in range(a.warmup):
        time_oracle(cfg, specs, weights, B, T_sample)
    times = []
    for _ in range(a.steps):
        dt, frames = time_oracle(cfg, specs, weights, B, T_sample)
        times.append(dt)
    tot = sum(times)
    value = frames * a.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "description": cfg.description,
                       "mode": specs[0].mode, "K": specs[0].K, "global_batch": cfg.B,
                       "T": cfg.T, "sample_batch": B, "sample_T": T_sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle",
                             "sample": f"{B} samples x T={T_sample} per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- training --
TRAIN_METRIC = "Conv-LIF training spike-frames/s (forward + surrogate-gradient BPTT backward)"


def run_train(a, cfg, rank, world, local, B_global):
    """One training step = the training forward of every layer (tac_conv_lif_forward_train,
    tac_or_pool2), a spike-count loss, and the backward of every layer
    (tac_conv_lif_backward, tac_or_pool2_backward); multi-GPU adds the NCCL all-reduce of
    the weight gradients (the data-parallel exchange step of training).  The paper's
    speedups are training speedups: the same step is timed
    for the dense per-timestep baseline, and the ratio is reported."""
    import torch
    import torch.distributed as dist
    from paper_2603_13810_b200 import configs, dist as D, network, tacsnn

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    b0, B = D.shard_range(B_global, world, rank)
    rate = cfg.inputs != "dvs"
    sg = dict(surrogate="fast_sigmoid", alpha=25.0, detach_reset=False) if rate else \
        dict(surrogate="arctan", alpha=2.0, detach_reset=True)          # App. E

    def build(mode, K):
        if a.whole_net:
            specs = configs.network_plan(cfg, mode=mode, K=K, B=B, engine=a.engine)
            weights = configs.network_weights(cfg)
        else:
            specs = configs.layer_plan(cfg, mode=mode, K=K, B=B, engine=a.engine)
            weights = configs.layer_weights(cfg)
        return network.TrainableNetwork(specs, weights, device=dev, **sg)

    x = tacsnn.pack(configs.make_inputs(cfg, B=B, b0=b0, device=dev))
    stream = torch.cuda.current_stream(dev)

    def timed(net):
        last = net.specs[-1]
        g = torch.Generator(device=dev).manual_seed(7 + rank)
        target = torch.zeros((B, last.C_out), device=dev)
        target[torch.arange(B, device=dev), torch.randint(0, last.C_out, (B,), generator=g, device=dev)] = 1.0

        def step():
            _, cnt, tape = net.forward_train(x)
            s_last = tape[-1][0]
            hc, wc = s_last.conv_hw
            T_out = tape[-1][4].shape[0]
            norm = float(T_out * hc * wc)
            # loss glue (user code): L = 0.5 sum (count / norm - target)^2  (spike-count readout)
            err = (cnt.float() / norm - target) / norm
            g_out = err[None, :, None, None, :].expand(T_out, B, hc, wc, s_last.C_out).contiguous()
            grads = net.backward(tape, g_out)
            if world > 1:   # data-parallel gradient exchange
                flat = torch.cat([torch.cat([r["g_weight"].reshape(-1), r["g_bias"]]) for r in grads])
                dist.all_reduce(flat)
            return grads

        launches = 0
        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / a.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    mode = a.mode or cfg.mode
    K = cfg.K if a.K is None else a.K
    net = build(mode, K)
    clocks = ClockSampler(local)
    clocks.start()
    ms = timed(net)
    clk = clocks.stop()
    engines = net.engines()
    del net
    ms_dense = timed(build("dense", 1))
    frames = B_global * cfg.T
    if rank == 0:
        line = {"metric": TRAIN_METRIC, "value": frames / (ms / 1e3), "unit": UNIT, "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": a.scaling, "vs_baseline": None, "dtype": "f32 gradients; forward as inference",
                "data": "synthetic",
                "config": {"workload": cfg.name + ("+FC" if a.whole_net else ""), "mode": mode, "K": K,
                           "global_batch": B_global, "per_rank_batch": B, "T": cfg.T,
                           "parallelism": f"dp{world}", "engines": engines, "surrogate": sg,
                           "loss": "0.5 sum (spike count / steps*pixels - one-hot)^2 (user glue)"},
                "dense_ms_per_step": ms_dense, "speedup_vs_dense": ms_dense / ms,
                "paper_context": "TAC training speedups 5.3-13.8x (M3 Max, MNIST K=4/8/16, P:255-257), "
                                 "5.1-13.1x (V100, P:331-337)",
                "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# -------------------------------------------------------------------- ours --
def launcher_check(a, rank, world):
    """Plumbing of the multi-rank bench on CPU (gloo): shard ranges and the output gather
    exactly as the GPU run uses them, one JSON line from rank 0 (tests/test_bench_launcher.py)."""
    import torch
    import torch.distributed as dist
    from paper_2603_13810_b200 import dist as D
    if world > 1:
        dist.init_process_group("gloo")
    B_global = a.B or 16
    b0, B = D.shard_range(B_global, world, rank)
    y = torch.arange(b0, b0 + B, dtype=torch.int32).reshape(1, B, 1).expand(2, B, 3).contiguous()
    cnt = torch.arange(b0, b0 + B, dtype=torch.int32).reshape(B, 1)
    if world > 1:
        y = D.gather_batch(y, dim=1)
        cnt = D.gather_batch(cnt, dim=0)
    ok = bool((y[0, :, 0] == torch.arange(B_global)).all()) and bool((cnt[:, 0] == torch.arange(B_global)).all())
    if rank == 0:
        print(json.dumps({"launcher_check": True, "n_gpus": world, "gpus_flag": a.gpus,
                          "global_batch": B_global, "per_rank_batch": B, "gather_ok": ok}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    ensure_ranks(a)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    from paper_2603_13810_b200 import configs
    cfg = configs.CONFIGS[a.config]
    B_global = a.B or cfg.B
    if a.scaling == "weak":
        B_global = B_global * world

    def specs_fn(B):
        return configs.layer_plan(cfg, mode=a.mode, K=a.K, B=B, engine=a.engine)

    if a.launcher_check:
        return launcher_check(a, rank, world)
    if a.train and a.impl != "reference":
        return run_train(a, cfg, rank, world, local, B_global)
    if a.impl == "reference":
        return run_reference(a, cfg, specs_fn, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2603_13810_b200 import dist as D, network, tacsnn

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    b0, B = D.shard_range(B_global, world, rank)
    specs = specs_fn(B)
    weights = configs.layer_weights(cfg)
    net = network.Network(specs, weights, device=dev)
    engines = net.engines()

    # inputs resident in HBM (larger than the 126 MB L2 for C5: no L2 flush needed)
    x_u8 = configs.make_inputs(cfg, B=B, b0=b0, device=dev)
    x = tacsnn.pack(x_u8)
    del x_u8
    def gather(y, cnt):
        """The path's only collective: final-layer packed spikes and counts."""
        if world > 1:
            D.gather_batch(y, dim=1)
            D.gather_batch(cnt, dim=0)

    def step(xin):
        y, counts, _, _ = net.forward(xin)
        gather(y, counts[-1])
        return y, counts

    launches_per_step = net.count_launches(x)
    for _ in range(a.warmup):
        step(x)
    torch.cuda.synchronize()

    # per-layer event timing inside the timed region (events on the launch stream)
    stream = torch.cuda.current_stream(dev)
    nL = len(specs)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(nL)] for _ in range(a.steps)]

    def step_timed(i, xin):
        B_ = xin.shape[1]
        cnt = None
        for li, (spec, prep) in enumerate(zip(net.specs, net.prepared)):
            s = spec if spec.B == B_ else spec.replace(B=B_)
            ev[i][li][0].record(stream)
            # the spike-count readout of the final layer only, as Network.forward
            xin, _, cnt = tacsnn.conv_lif(s, prep, xin, want_counts=(li == nL - 1))
            ev[i][li][1].record(stream)
        gather(xin, cnt)
        return xin

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(a.steps):
        step_timed(i, x)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_local = t_start.elapsed_time(t_end)
    ms_t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_total = float(ms_t.item())
    ms_per_step = ms_total / a.steps
    layer_ms = [statistics.mean(ev[i][li][0].elapsed_time(ev[i][li][1]) for i in range(a.steps))
                for li in range(nL)]

    frames_per_step = B_global * cfg.T
    value = frames_per_step / (ms_per_step / 1e3)

    # ---------------- end to end: pinned host input -> device -> counts back
    # Every step copies its whole packed input from pinned host memory (on a copy
    # stream, double-buffered so the copy of step i+1 overlaps the forward of step i)
    # and reads its spike-count readout back to the host.
    e2e = None
    if not a.no_e2e:
        host_x = torch.empty(x.shape, dtype=torch.int32, pin_memory=True)
        host_x.copy_(x)
        bufs = [torch.empty_like(x), torch.empty_like(x)]
        host_cnt = torch.empty((B, specs[-1].C_out), dtype=torch.int32, pin_memory=True)
        copy_stream = torch.cuda.Stream(dev)
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        freed = [torch.cuda.Event(), torch.cuda.Event()]

        def e2e_steps(n):
            copy_stream.wait_stream(stream)
            with torch.cuda.stream(copy_stream):
                bufs[0].copy_(host_x, non_blocking=True)
                copied[0].record(copy_stream)
            for i in range(n):
                j = i % 2
                if i + 1 < n:
                    jn = (i + 1) % 2
                    with torch.cuda.stream(copy_stream):
                        if i >= 1:
                            copy_stream.wait_event(freed[jn])   # step i-1 is done with it
                        bufs[jn].copy_(host_x, non_blocking=True)
                        copied[jn].record(copy_stream)
                stream.wait_event(copied[j])
                _, c = step(bufs[j])
                freed[j].record(stream)
                host_cnt.copy_(c[-1], non_blocking=True)

        e2e_steps(2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_steps(a.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": frames_per_step / (float(e_ms.item()) / a.steps / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(host_x.numel() * 4 * world),
               "d2h_bytes_per_step": int(host_cnt.numel() * 4 * world)}
        del host_x, bufs

    # ---------------- roofline of the dominant kernel (per-layer launch)
    peaks = load_peaks()
    flops = useful_flops_per_sample(specs)
    nsteps_ps = neuron_steps_per_sample(specs)
    bytes_ = algorithmic_bytes_per_sample(specs)
    long_run = a.steps * ms_per_step > 2000
    tensor_peak = (peaks["bf16_sustained"] if long_run else peaks["bf16"]) * 2.0  # int8 = bf16 x 2
    alu_peak = 148 * 128 * peaks["sm_max_mhz"] * 1e6 / 1e12  # T lane-ops/s
    traffic = load_traffic()
    layer_rows = []
    for li in range(nL):
        dur = layer_ms[li] / 1e3
        t_ach = flops[li] * B / dur / 1e12
        a_ach = LIF_ALG_OPS * nsteps_ps[li] * B / dur / 1e12
        row = {"layer": li, "engine": engines[li], "ms": layer_ms[li],
               "useful_tflops": t_ach,
               "tensor_frac": t_ach / tensor_peak if engines[li] == "tcgen05" else None,
               "tensor_issued_frac": 2.0 * t_ach / tensor_peak if engines[li] == "tcgen05" else None,
               "lif_tops": a_ach, "alu_frac": a_ach / alu_peak,
               "packed_gbs": bytes_[li] * B / dur / 1e9,
               "frames_per_s": B * specs[li].T / dur}
        layer_rows.append(row)
    dom = max(range(nL), key=lambda li: layer_ms[li])
    dspec, drow = specs[dom], layer_rows[dom]
    tkey = f"{cfg.name}/{specs[0].mode}/K{specs[0].K}/B{B}/layer{dom}"
    if engines[dom] == "tcgen05" and (drow["tensor_frac"] or 0) >= drow["alu_frac"]:
        roof = {"bound": "tensor", "achieved": drow["useful_tflops"], "peak": tensor_peak,
                "unit": "TFLOP/s", "frac": drow["tensor_frac"],
                "peak_note": f"int8 tcgen05 peak = {peaks['source']} bf16 x 2 (nominal 4.5/2.25); "
                             f"achieved = useful conv FLOPs (2 int8 weight slices issue 2x)"}
    else:
        roof = {"bound": "alu", "achieved": drow["lif_tops"], "peak": alu_peak,
                "unit": "Tops/s", "frac": drow["alu_frac"],
                "peak_note": "148 SM x 128 lanes x SM clock (one 32-lane warp instr/cycle/SMSP); "
                             f"achieved = {LIF_ALG_OPS:.0f} algorithmic LIF ops per neuron-step "
                             "(FMA, compare, reset subtract)"}
    roof["traffic"] = traffic.get(tkey)
    roof["kernel"] = f"layer {dom} ({dspec.C_in}->{dspec.C_out} @{dspec.H}x{dspec.W}, {engines[dom]})"
    roof["hbm_achieved_gbs"] = drow["packed_gbs"]

    # "% tensor-pipe peak" of the metric, for the DVS128-shaped 128->128 conv (layer 1, the
    # north star's tensor-pipe target): useful conv FLOP/s against the measured dense bf16 peak
    # (the precision the paper's fp16/fp32 conv runs in) and issued int8 ops (two weight slices)
    # against the int8 peak derived from it; the direct ncu tensor-pipe activity is in profiles/.
    tensor_pipe = None
    tl = 1 if nL > 1 and engines[1] == "tcgen05" else None
    if tl is not None:
        u = layer_rows[tl]["useful_tflops"]
        bf16 = peaks["bf16_sustained"] if long_run else peaks["bf16"]
        tensor_pipe = {"layer": tl, "useful_tflops": u, "issued_int8_tops": 2.0 * u,
                       "useful_vs_measured_bf16_peak": u / bf16,
                       "issued_vs_derived_int8_peak": 2.0 * u / tensor_peak,
                       "issued_vs_nominal_int8_peak": 2.0 * u / 4500.0,
                       "note": "int8 operands beat the measured cuBLAS bf16 rate (72 % of nominal), so "
                               "the derived int8 peak (measured bf16 x 2) is below what int8 issues; "
                               "nominal dense int8 = 4.5 POPS",
                       "ncu_tensor_active": "profiles/ncu_c5_layer1_r02.txt (sm__pipe_tensor_cycles_active)"}

    # ---------------- v_final on: every layer also writes its fp32 membrane state
    # (SURVEY.md 8(d) "measure with and without it"); a few extra steps after the timed region
    vfinal = None
    if not a.no_v_final:
        nvf = max(2, min(a.steps, 5))
        for _ in range(1):
            net.forward(x, want_v_final=True)
        torch.cuda.synchronize()
        v0e, v1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0e.record(stream)
        for _ in range(nvf):
            net.forward(x, want_v_final=True)
        v1e.record(stream)
        torch.cuda.synchronize()
        vms = v0e.elapsed_time(v1e) / nvf
        vbytes = sum(4.0 * s_.B * s_.conv_hw[0] * s_.conv_hw[1] * s_.C_out for s_ in specs)
        vfinal = {"ms_per_step": vms, "value": frames_per_step / (vms / 1e3),
                  "v_final_bytes_per_step": vbytes, "steps": nvf,
                  "note": "rank-local: every layer writes fp32 v_final [B,H',W',C_out]"}

    # ---------------- the whole network: the FC head (+ VotingLayer for DVS) on the stack's
    # output, timed the same way after the main region
    whole = None
    if not a.no_head:
        nconv = len(cfg.layers)
        hspecs = configs.network_plan(cfg, mode=a.mode, K=a.K, B=B, engine=a.engine)[nconv:]
        head = network.Network(hspecs, configs.network_weights(cfg)[nconv:], device=dev,
                               voters=configs.VOTERS[configs.head_kind(cfg)])
        y0, _, _, _ = net.forward(x)

        def head_step():
            _, hc, _, _ = head.forward(y0)
            return head.readout(hc[-1])
        head_step()
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nh = max(3, min(a.steps, 10))
        h0.record(stream)
        for _ in range(nh):
            head_step()
        h1.record(stream)
        torch.cuda.synchronize()
        hms = h0.elapsed_time(h1) / nh
        whole = {"head_ms_per_step": hms, "ms_per_step": ms_per_step + hms,
                 "value": frames_per_step / ((ms_per_step + hms) / 1e3),
                 "head": " -> ".join(f"FC({s_.C_in}->{s_.C_out})" for s_ in hspecs) +
                         (f" -> VotingLayer({head.voters})" if head.voters else " -> spike counts"),
                 "head_engines": head.engines(),
                 "note": "rank-local head after the timed conv stack; value = B*T / (stack + head)"}
        del head, y0

    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        cpu = cpu_baseline(cfg, specs, weights, a.cpu_sample_T)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
            "dtype": dtype_note(specs, engines),
            "data": "synthetic",
            "config": {"workload": cfg.name, "description": cfg.description,
                       "mode": specs[0].mode, "K": specs[0].K, "global_batch": B_global,
                       "per_rank_batch": B, "T": cfg.T, "parallelism": f"dp{world}",
                       "layers": len(specs), "engines": engines,
                       "l2": l2_note(specs, B)},
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": launches_per_step * a.steps,
            "roofline": roof,
            "tensor_pipe": tensor_pipe,
            "cpu_baseline": cpu,
            "v_final_on": vfinal,
            "whole_network": whole,
            "layers": layer_rows,
            "peaks": peaks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
