"""Seeded synthetic inputs shaped like the paper's workloads (no method arithmetic).

Every generator is a counter-based integer hash of (seed, global sample index,
coordinates), computed with int64 torch ops that are bit-identical on CPU and
CUDA.  So the same sample is the same tensor whichever device, batch shard or
chunk produces it -- the CUDA path and the oracle get identical spikes, and a
parity test can regenerate any single sample of a full-size batch.

Workload recipes:
  * bernoulli(rho): i.i.d. spikes, config C1 ("rate-coded Poisson spikes rho=0.1",
    read as Bernoulli per step, R8).
  * mnist / fmnist: rate coding (S_t ~ Bernoulli(I)) of synthetic
    intensity maps -- 'mnist': 2 hollow elliptical strokes (mean ~0.13, the
    MNIST pixel mean); 'fmnist': one filled textured silhouette (mean ~0.29).
  * dvs: DVS128-Gesture-like binary event-occurrence frames [T,B,2,H,W]
    (PAPER.md:231, 601-604): 1-2 disks (r 12-24 px at 128^2) moving 3-8 px/bin
    in a class-dependent direction, bouncing off the borders; ON (channel 1)
    marks newly covered pixels, OFF (channel 0) newly uncovered ones, each with
    probability 0.8, plus 0.002 noise per (polarity, pixel, bin).
Weights: N(0, (gain / sqrt(C_in R S))^2) from a seeded torch CPU generator;
bias U(-0.1, 0.1) (stands in for folded BN, R3).
"""
from __future__ import annotations

import torch

M32 = 0xFFFFFFFF
P24 = 1 << 24


def _mix(x: torch.Tensor) -> torch.Tensor:
    """32-bit integer finaliser on int64 tensors holding values in [0, 2^32)."""
    x = ((x ^ (x >> 16)) * 0x45D9F3B) & M32
    x = ((x ^ (x >> 16)) * 0x45D9F3B) & M32
    return x ^ (x >> 16)


def _h(h: torch.Tensor, v) -> torch.Tensor:
    return _mix((h * 0x01000193 + v + 0x9E3779B9) & M32)


def _sample_params(seed: int, b_idx: torch.Tensor, n: int) -> torch.Tensor:
    """n independent 32-bit draws per sample: int64 [B, n]."""
    h = _h(torch.full_like(b_idx, seed & M32), b_idx)
    k = torch.arange(n, device=b_idx.device, dtype=torch.int64)
    return _h(h[:, None], k[None, :] * 7919)


def _uniform_int(draw: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    """integer in [lo, hi] from a 32-bit draw."""
    return lo + draw % (hi - lo + 1)


def _bernoulli_from(key: torch.Tensor, thr24: torch.Tensor) -> torch.Tensor:
    return ((key & (P24 - 1)) < thr24).to(torch.uint8)


def _frame_keys(seed, t, b_idx, C, H, W, salt=0):
    dev = b_idx.device
    c = torch.arange(C, device=dev, dtype=torch.int64)
    y = torch.arange(H, device=dev, dtype=torch.int64)
    x = torch.arange(W, device=dev, dtype=torch.int64)
    h = _h(torch.full_like(b_idx, (seed * 31 + salt) & M32), b_idx)        # [B]
    h = _h(h, t * 104729)
    h = _h(h[:, None], c[None, :] * 15485863)                              # [B, C]
    h = _h(h[:, :, None], y[None, None, :] * 32452843)                     # [B, C, H]
    return _h(h[..., None], x[None, None, None, :])                        # [B, C, H, W]


def _b_idx(B, b0, device):
    return torch.arange(b0, b0 + B, device=device, dtype=torch.int64)


def intensity(kind: str, seed: int, B: int, H: int = 28, W: int = 28, b0: int = 0,
              device="cpu") -> torch.Tensor:
    """Synthetic intensity maps, int64 in [0, 255], shape [B, 1, H, W]."""
    b_idx = _b_idx(B, b0, device)
    yy = torch.arange(H, device=device, dtype=torch.int64)[None, :, None]
    xx = torch.arange(W, device=device, dtype=torch.int64)[None, None, :]
    img = torch.zeros((B, H, W), dtype=torch.int64, device=device)
    if kind == "mnist":
        p = _sample_params(seed, b_idx, 16)
        for s in range(2):                              # two hollow elliptical strokes
            cx = _uniform_int(p[:, 8 * s + 0], 8, W - 9)[:, None, None]
            cy = _uniform_int(p[:, 8 * s + 1], 8, H - 9)[:, None, None]
            rx = _uniform_int(p[:, 8 * s + 2], 3, 7)[:, None, None]
            ry = _uniform_int(p[:, 8 * s + 3], 4, 9)[:, None, None]
            th = _uniform_int(p[:, 8 * s + 4], 1, 2)[:, None, None]
            dx, dy = xx - cx, yy - cy
            outer = (dx * ry) ** 2 + (dy * rx) ** 2 <= (rx * ry) ** 2
            rxi, ryi = (rx - th).clamp(min=1), (ry - th).clamp(min=1)
            inner = (dx * ryi) ** 2 + (dy * rxi) ** 2 < (rxi * ryi) ** 2
            ring = outer & ~inner
            img = torch.maximum(img, ring.to(torch.int64) * 255)
    elif kind == "fmnist":
        p = _sample_params(seed, b_idx, 8)
        x0 = _uniform_int(p[:, 0], 4, 9)[:, None, None]
        x1 = _uniform_int(p[:, 1], 18, 23)[:, None, None]
        y0 = _uniform_int(p[:, 2], 3, 7)[:, None, None]
        y1 = _uniform_int(p[:, 3], 18, 24)[:, None, None]
        inside = (xx >= x0) & (xx <= x1) & (yy >= y0) & (yy <= y1)
        tex = 128 + _mix((p[:, 4][:, None, None] + yy * 131 + xx * 7) & M32) % 128
        img = inside.to(torch.int64) * tex
    else:
        raise ValueError(kind)
    return img[:, None]


def rate_coded(kind: str, seed: int, T: int, B: int, H: int = 28, W: int = 28, b0: int = 0,
               rho: float = 0.1, device="cpu") -> torch.Tensor:
    """u8 spikes [T, B, 1, H, W]: S_t ~ Bernoulli(I) per pixel and step.
    kind 'bernoulli' uses the constant rate rho (config C1)."""
    b_idx = _b_idx(B, b0, device)
    if kind == "bernoulli":
        thr = torch.full((B, 1, H, W), int(round(rho * P24)), dtype=torch.int64, device=device)
    else:
        thr = (intensity(kind, seed, B, H, W, b0, device) * P24) // 255
    out = torch.empty((T, B, 1, H, W), dtype=torch.uint8, device=device)
    for t in range(T):
        out[t] = _bernoulli_from(_frame_keys(seed, t, b_idx, 1, H, W, salt=1), thr)
    return out


def _disk_centre(p0, v, r, t, size):
    """Bouncing 1-D position: triangle wave over [r, size-1-r]."""
    L = (size - 1 - 2 * r).clamp(min=1)
    q = torch.remainder(p0 - r + v * t, 2 * L)
    return r + torch.where(q <= L, q, 2 * L - q)


def dvs_events(seed: int, T: int, B: int, H: int = 128, W: int = 128, b0: int = 0,
               device="cpu", noise: float = 0.002, p_event: float = 0.8) -> torch.Tensor:
    """u8 binary event-occurrence frames [T, B, 2, H, W] (channel 0 OFF, 1 ON)."""
    b_idx = _b_idx(B, b0, device)
    p = _sample_params(seed, b_idx, 16)
    cls = p[:, 0] % 11                                   # 11 gesture classes
    dirs = torch.tensor([[1, 0], [-1, 0], [0, 1], [0, -1], [1, 1], [-1, -1], [1, -1], [-1, 1],
                         [2, 1], [-1, 2], [1, -2]], dtype=torch.int64, device=device)
    d = dirs[cls]                                        # [B, 2]
    ndisk = 1 + (p[:, 1] % 2)                            # 1 or 2 disks
    yy = torch.arange(H, device=device, dtype=torch.int64)[None, :, None]
    xx = torch.arange(W, device=device, dtype=torch.int64)[None, None, :]
    disks = []
    for k in range(2):
        r = _uniform_int(p[:, 2 + 5 * k], 12 * H // 128, 24 * H // 128).clamp(min=2)
        speed = _uniform_int(p[:, 3 + 5 * k], 3, 8)
        sgn = 1 - 2 * k                                  # second disk moves the other way
        vx, vy = sgn * speed * d[:, 0], sgn * speed * d[:, 1]
        x0 = _uniform_int(p[:, 4 + 5 * k], 0, W - 1)
        y0 = _uniform_int(p[:, 5 + 5 * k], 0, H - 1)
        active = (ndisk > k)
        disks.append((r, vx, vy, x0, y0, active))

    def covered(t):
        cov = torch.zeros((B, H, W), dtype=torch.bool, device=device)
        for r, vx, vy, x0, y0, active in disks:
            cx = _disk_centre(x0, vx, r, t, W)[:, None, None]
            cy = _disk_centre(y0, vy, r, t, H)[:, None, None]
            rr = r[:, None, None]
            cov |= ((xx - cx) ** 2 + (yy - cy) ** 2 <= rr * rr) & active[:, None, None]
        return cov

    thr_ev = int(round(p_event * P24))
    thr_noise = int(round(noise * P24))
    out = torch.empty((T, B, 2, H, W), dtype=torch.uint8, device=device)
    prev = covered(-1)
    for t in range(T):
        cur = covered(t)
        keys = _frame_keys(seed, t, b_idx, 2, H, W, salt=2)
        ev_ok = (keys & (P24 - 1)) < thr_ev
        nz = ((keys >> 8) & (P24 - 1)) < thr_noise
        on = (cur & ~prev) & ev_ok[:, 1]
        off = (prev & ~cur) & ev_ok[:, 0]
        out[t, :, 1] = (on | nz[:, 1]).to(torch.uint8)
        out[t, :, 0] = (off | nz[:, 0]).to(torch.uint8)
        prev = cur
    return out


def dvs_log_counts(seed: int, T: int, B: int, H: int = 128, W: int = 128, b0: int = 0,
                   device="cpu", sub: int = 4) -> torch.Tensor:
    """Continuous-valued DVS-like input (the paper's first-layer input is log-normalised
    event counts): each of the T bins sums `sub` consecutive event-
    occurrence frames of dvs_events, then x = log(1 + count) / log(1 + sub) in [0, 1].
    fp32 [T, B, 2, H, W]."""
    ev = dvs_events(seed, T * sub, B, H, W, b0=b0, device=device)
    cnt = ev.view(T, sub, B, 2, H, W).sum(dim=1, dtype=torch.int32).to(torch.float64)
    return (torch.log1p(cnt) / torch.log1p(torch.tensor(float(sub), dtype=torch.float64))).to(torch.float32)


def weights(seed: int, C_out: int, C_in: int, R: int = 3, S: int = 3, gain: float = 1.0):
    """fp32 [C_out, C_in, R, S] ~ N(0, (gain/sqrt(C_in R S))^2) and bias U(-0.1, 0.1)."""
    g = torch.Generator().manual_seed(seed)
    w = torch.randn((C_out, C_in, R, S), generator=g, dtype=torch.float64)
    w = (w * (gain / (C_in * R * S) ** 0.5)).to(torch.float32)
    b = ((torch.rand((C_out,), generator=g, dtype=torch.float64) * 0.2) - 0.1).to(torch.float32)
    return w, b
