"""§8 row f1: the bulk-synchronous baseline (separate kernels + all-to-all, bulksync.py) computes the
reference's layer (oracle.hpp:44-120) -- on CPU tensors here, world 1 and world 2 over gloo; bench.py
times the same code on the GPU with NCCL."""
import multiprocessing as mp
import socket

import numpy as np
import torch

import paper_2506_04667_b200 as fd
from oracle import pyoracle as po
from paper_2506_04667_b200.bulksync import BulkSyncMoE


def _close(got, want):
    err = np.abs(got.astype(np.float64) - want)
    assert np.all(err <= 1e-4 + 1e-3 * np.abs(want)), float(err.max())


def test_bulksync_world1_matches_oracle():
    cfg = fd.MoeConfig(tokens_per_device=192, embed_dim=64, ffn_dim=128, experts_total=8, devices=1, topk=2, seed=5)
    model, shard = fd.make_model(cfg), fd.make_shards(cfg)[0]
    got = BulkSyncMoE(cfg, model, device="cpu").forward(torch.from_numpy(shard)).numpy()
    _close(got, po.dense_forward(shard, model, cfg))


def test_bulksync_world2_gloo_matches_oracle():
    import dist_workers
    world = 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=dist_workers.run_bulksync, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = fd.MoeConfig(tokens_per_device=128, embed_dim=64, ffn_dim=96, experts_total=8, devices=world, topk=2,
                       seed=3)
    model = fd.make_model(cfg)
    for r, shard in enumerate(fd.make_shards(cfg)):
        _close(got[r], po.dense_forward(shard, model, cfg))
