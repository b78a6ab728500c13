"""World-size-2 CPU test of the data-parallel path (gloo): each rank owns a
contiguous batch shard, runs the layer (the CPU oracle stands in for the per-rank
CUDA compute, which cannot run here), and the gathered packed spikes / counts
must equal the single-process full-batch result bit for bit (P13: samples are
independent, the batch split is invisible)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O
        from paper_2603_13810_b200 import configs, dist as D
        cfg = configs.CONFIGS["C4"]
        B = 4
        b0, n = D.shard_range(B, world, rank)
        S = configs.make_inputs(cfg, B=n, b0=b0, T=4).numpy()   # rank generates its own shard
        w, b = configs.layer_weights(cfg)[0]
        r = O.forward(S[:, :, :, :32, :32], w.numpy(), b.numpy(), K=2, mode="tactp", beta=0.5, pad=1)
        spk = torch.from_numpy(O.pack_spikes(O.or_pool2(r["out"])).view(np.int32))  # [T,n,H,WPR]
        cnt = torch.from_numpy(r["counts"].astype(np.int32))                        # [n,C]
        full_spk = D.gather_batch(spk, dim=1)
        full_cnt = D.gather_batch(cnt, dim=0)
        if rank == 0:
            np.savez(result_path, spk=full_spk.numpy(), cnt=full_cnt.numpy())
    finally:
        dist.destroy_process_group()


def test_world2_gather_equals_single_process(tmp_path):
    from oracle import oracle as O
    from paper_2603_13810_b200 import configs
    O.build()
    world, port = 2, _free_port()
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, port, path), nprocs=world, join=True)
    got = np.load(path)
    cfg = configs.CONFIGS["C4"]
    S = configs.make_inputs(cfg, B=4, T=4).numpy()
    w, b = configs.layer_weights(cfg)[0]
    r = O.forward(S[:, :, :, :32, :32], w.numpy(), b.numpy(), K=2, mode="tactp", beta=0.5, pad=1)
    ref_spk = O.pack_spikes(O.or_pool2(r["out"])).view(np.int32)
    assert r["out"].sum() > 0
    assert np.array_equal(got["spk"], ref_spk)
    assert np.array_equal(got["cnt"], r["counts"].astype(np.int32))


def test_shard_range():
    from paper_2603_13810_b200 import dist as D
    assert D.shard_range(2048, 8, 3) == (768, 256)
    with pytest.raises(ValueError):
        D.shard_range(10, 4, 0)
