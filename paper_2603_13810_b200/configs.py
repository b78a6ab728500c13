"""The five BASELINE.json workloads (configs C1-C5) as stacks of Conv-LIF layers.

Architectures follow PAPER.md:234-235; layer_plan is the conv blocks, network_plan the
whole network with its FC head (see below):
  MNIST/FMNIST: Conv(1->32,3,pad 0)->LIF->Pool(2)->Conv(32->64,3,pad 0)->LIF
                (pad 0 from FC(1600)=64*5*5; the odd 11x11
                output of layer 2 is left unpooled, reading D13)
  DVS128:       5 x {Conv(128,3,pad 1)->LIF->MaxPool(2)} on 2x128x128 events
BN is folded into the bias (reading R3); MaxPool of binary spikes is the fused
OR-pool.  beta = 0.9 (rate-coded) / 0.5 (DVS), v_th = 1, subtract reset
(App. E).  Cascaded TAC uses K_l = min(K, T_l) and
T_{l+1} = T_l / K_l (App. B, reading D7).
"""
from __future__ import annotations

import dataclasses

from . import synth

# Per-layer weight gains (synth.weights), calibrated once with the oracle so that
# every layer fires at roughly 5-25 % in the config's primary mode
# (scripts/calibrate_gains.py); frozen here.
GAINS = {
    "mnist": [0.78, 0.46],
    "mnist_fc": [2.0, 2.0],   # FC(1600->128), FC(128->10) of the whole network (set below)
    "dvs": [7.1, 1.08, 1.01, 1.01, 0.89],
    "dvs_fc": [0.81, 1.48],   # FC(2048->512), FC(512->110) of the DVS network (--head, C4 B=2)
}


@dataclasses.dataclass(frozen=True)
class LayerCfg:
    C_in: int
    C_out: int
    H: int
    W: int
    pad: int
    pool: int


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    description: str
    T: int
    B: int
    K: int
    mode: str                 # primary mode: "tac" | "tactp" | "dense"
    beta: float
    inputs: str               # synth generator: bernoulli | mnist | fmnist | dvs
    layers: tuple
    gains: tuple
    seeds: tuple
    compare: tuple = ("dense",)   # other modes the config is reported against

    @property
    def C_in(self):
        return self.layers[0].C_in

    @property
    def H(self):
        return self.layers[0].H

    @property
    def W(self):
        return self.layers[0].W


_MNIST = (LayerCfg(1, 32, 28, 28, 0, 2), LayerCfg(32, 64, 13, 13, 0, 1))
_DVS = (LayerCfg(2, 128, 128, 128, 1, 2), LayerCfg(128, 128, 64, 64, 1, 2),
        LayerCfg(128, 128, 32, 32, 1, 2), LayerCfg(128, 128, 16, 16, 1, 2),
        LayerCfg(128, 128, 8, 8, 1, 2))

CONFIGS = {
    "C1": Config("C1", "single Conv-LIF layer 1->8 ch 3x3, 28x28 rate-coded Poisson spikes "
                 "(rho=0.1), T=8, K=4, batch 4, TAC vs dense",
                 T=8, B=4, K=4, mode="tac", beta=0.9, inputs="bernoulli",
                 layers=(LayerCfg(1, 8, 28, 28, 0, 1),), gains=(1.42,), seeds=(0, 1, 2)),
    "C2": Config("C2", "MNIST-shaped 2-layer conv SNN (1->32->64 ch 3x3), T=16, K=2/4/8, "
                 "batch 256, TAC collapse",
                 T=16, B=256, K=4, mode="tac", beta=0.9, inputs="mnist", layers=_MNIST,
                 gains=tuple(GAINS["mnist"]), seeds=(0, 1, 2)),
    "C3": Config("C3", "Fashion-MNIST-shaped conv SNN, T=32, K=8, batch 1024, TAC vs dense "
                 "per-timestep baseline",
                 T=32, B=1024, K=8, mode="tac", beta=0.9, inputs="fmnist", layers=_MNIST,
                 gains=tuple(GAINS["mnist"]), seeds=(0, 1, 2)),
    "C4": Config("C4", "DVS128-Gesture-shaped synthetic events 2x128x128, T=16, K=2, batch 64, "
                 "TAC-TP (K LIF steps share conv output)",
                 T=16, B=64, K=2, mode="tactp", beta=0.5, inputs="dvs", layers=_DVS,
                 gains=tuple(GAINS["dvs"]), seeds=(0, 42, 123), compare=("dense", "tac")),
    "C5": Config("C5", "DVS128-shaped TAC-TP, T=32, K=4, batch 2048 batch-sharded across "
                 "1/2/4/8 B200",
                 T=32, B=2048, K=4, mode="tactp", beta=0.5, inputs="dvs", layers=_DVS,
                 gains=tuple(GAINS["dvs"]), seeds=(0, 42, 123)),
}


def layer_plan(cfg: Config, mode: str | None = None, K: int | None = None, B: int | None = None,
               engine: str = "auto", T: int | None = None):
    """LayerSpecs of the stack (imports the binding lazily).  With T not a multiple of
    K (the paper's T = 25) the layers use a partial last group (reading D6') and a TAC
    layer passes ceil(T_l / K_l) steps on."""
    from .tacsnn import LayerSpec
    mode = mode or cfg.mode
    K = cfg.K if K is None else K
    B = cfg.B if B is None else B
    specs, t = [], cfg.T if T is None else T
    for L in cfg.layers:
        Kl = 1 if mode == "dense" else min(K, t)
        specs.append(LayerSpec(T=t, B=B, C_in=L.C_in, H=L.H, W=L.W, C_out=L.C_out, R=3, S=3,
                               stride=1, pad=L.pad, K=Kl, mode=mode, beta=cfg.beta, v_th=1.0,
                               v_reset=0.0, reset="subtract", out_pool=L.pool, engine=engine,
                               partial=(t % Kl != 0)))
        if mode == "tac":
            t = -(-t // Kl)
    return specs


# Mode-specific gains: the DVS stack run DENSE (one LIF step per frame with beta = 0.5
# and the sparse event input) goes nearly silent in its deep layers with the TAC-TP
# gains, which would make deep-layer parity vacuous; these are calibrated the same way
# in dense mode (scripts/calibrate_gains.py C4 --mode dense [--head]).
MODE_GAINS = {
    ("dvs", "dense"): (15.49, 1.59, 1.59, 1.49, 1.31),   # C4 --mode dense, B=2: each layer ~10 %
    ("dvs_fc", "dense"): (1.18, 2.34),                   # C4 --mode dense --head
    ("dvs", "tac"): (11.19, 1.4, 1.49, 1.4, 1.81),        # C4 --mode tac (K = 2 cascade)
}


def gains_for(cfg: Config, mode: str | None = None):
    g = MODE_GAINS.get((head_kind(cfg), mode or cfg.mode))
    return tuple(g) if g else cfg.gains


def layer_weights(cfg: Config, seed: int | None = None, mode: str | None = None):
    """Seeded weights of the conv stack; `mode` selects mode-specific gains (MODE_GAINS)."""
    seed = cfg.seeds[0] if seed is None else seed
    out = []
    for i, (L, g) in enumerate(zip(cfg.layers, gains_for(cfg, mode))):
        out.append(synth.weights(seed * 1000 + i, L.C_out, L.C_in, 3, 3, gain=g))
    return out


def make_inputs(cfg: Config, B: int | None = None, b0: int = 0, seed: int | None = None,
                T: int | None = None, device="cpu"):
    """u8 spikes [T, B, C_in, H, W] for samples b0 .. b0+B-1 of the config."""
    seed = cfg.seeds[0] if seed is None else seed
    B = cfg.B if B is None else B
    T = cfg.T if T is None else T
    if cfg.inputs == "dvs":
        return synth.dvs_events(seed, T, B, cfg.H, cfg.W, b0=b0, device=device)
    return synth.rate_coded(cfg.inputs, seed, T, B, cfg.H, cfg.W, b0=b0, rho=0.1, device=device)


def conv_calls(cfg: Config, mode: str | None = None, K: int | None = None, T: int | None = None) -> int:
    """Logical conv calls of the stack per sample: sum_l ceil(T_l / K_l)."""
    return sum(-(-s.T // (1 if s.mode == "dense" else s.K)) for s in layer_plan(cfg, mode, K, B=1, T=T))


# --- whole networks: conv stack + FC head ----------------------
# MNIST/FMNIST: Conv(1->32)->LIF->Pool(2)->Conv(32->64)->LIF->Pool(2) [11x11 -> 5x5,
#   floor] ->FC(1600->128)->LIF->FC(128->10)->LIF; readout = the final
#   layer's spike counts ("LIF + spike count").
# DVS: 5 x {Conv(128)->LIF->MaxPool(2)} ->FC(->512)->LIF->FC(512->110)->LIF->VotingLayer
#   (10 voters, 11 classes; FC widths SURVEY.md App. A 7).  At the
#   paper's 64x64 input the flattened map is 2x2x128 = 512; the BASELINE configs'
#   128x128 input gives 4x4x128 = 2048 (reading D14).  The VotingLayer averages the
#   firing rates of each class's 10 voters (tac_vote).
# The FC layers are 1x1 "convolutions" of a 1x1 image (C_in = flattened map), TAC-
# aggregated like the convs (they are linear too) and run on the tcgen05 FC kernel.
HEADS = {"mnist": (128, 10), "dvs": (512, 110)}
VOTERS = {"mnist": None, "dvs": 10}


def head_kind(cfg: Config) -> str:
    return "dvs" if cfg.inputs == "dvs" else "mnist"


def _flat_in(cfg: Config) -> int:
    h, w = cfg.H, cfg.W
    for L in cfg.layers:
        h, w = h + 2 * L.pad - 2, w + 2 * L.pad - 2
        if L.pool == 2 or cfg.inputs != "dvs":   # MNIST pools both blocks (layer 2 floor 11 -> 5)
            h, w = h // 2, w // 2
    return h * w * cfg.layers[-1].C_out


def head_dims(cfg: Config):
    """((C_in, C_out) of FC 1, (C_in, C_out) of FC 2)."""
    h1, h2 = HEADS[head_kind(cfg)]
    return ((_flat_in(cfg), h1), (h1, h2))


def network_plan(cfg: Config, mode: str | None = None, K: int | None = None, B: int | None = None,
                 engine: str = "auto", T: int | None = None):
    from .tacsnn import LayerSpec
    convs = layer_plan(cfg, mode=mode, K=K, B=B, engine=engine, T=T)
    if head_kind(cfg) == "mnist":
        convs[1] = convs[1].replace(out_pool=2)        # 11x11 -> 5x5 (floor)
    mode = mode or cfg.mode
    K = cfg.K if K is None else K
    last = convs[-1]
    t = last.T if mode != "tac" else -(-last.T // last.K)
    specs = list(convs)
    for c_in, c_out in head_dims(cfg):
        Kl = 1 if mode == "dense" else min(K, t)
        specs.append(LayerSpec(T=t, B=convs[0].B, C_in=c_in, H=1, W=1, C_out=c_out, R=1, S=1,
                               stride=1, pad=0, K=Kl, mode=mode, beta=cfg.beta, v_th=1.0,
                               v_reset=0.0, reset="subtract", out_pool=1, engine=engine,
                               partial=(t % Kl != 0)))
        if mode == "tac":
            t = -(-t // Kl)
    return specs


def network_weights(cfg: Config, seed: int | None = None, mode: str | None = None):
    seed = cfg.seeds[0] if seed is None else seed
    w = layer_weights(cfg, seed, mode)
    fc = MODE_GAINS.get((head_kind(cfg) + "_fc", mode or cfg.mode)) or GAINS[head_kind(cfg) + "_fc"]
    for i, ((c_in, c_out), g) in enumerate(zip(head_dims(cfg), fc)):
        w.append(synth.weights(seed * 1000 + 10 + i, c_out, c_in, 1, 1, gain=g))
    return w
