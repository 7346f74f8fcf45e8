"""Worker bodies for tests/test_dist_cpu.py (imported by spawned gloo ranks)."""
import os

import numpy as np


def run(rank: int, world: int, port: int, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_04667_b200 as fd
        from paper_2506_04667_b200 import dist as fdist
        from oracle import pyoracle as po
        res = {}
        # heap-blob exchange: rank-major, byte-exact
        blob = bytes([rank]) * 64 + b"heap"
        res["blobs"] = fdist.exchange_blobs(blob)
        # latency reduce
        res["max"] = fdist.max_over_ranks(1.0 + rank * 0.25)
        # per-rank routing -> the reference's P x P bytes matrix
        cfg = fd.MoeConfig(tokens_per_device=256, embed_dim=64, ffn_dim=64, experts_total=8, devices=world,
                           topk=2, seed=4)
        model = fd.make_model(cfg)
        shard = fdist.rank_shards(cfg, [rank])[0]
        g = po.gate(shard, model.wg, cfg.topk, fd.expert_capacity(cfg))
        res["payload"] = fdist.gather_payload(cfg, g["slot_counts"])
        res["experts"] = list(fdist.rank_experts(cfg, rank))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def run_bulksync(rank: int, world: int, port: int, q):
    """One rank of the bulk-synchronous baseline (bulksync.py) over gloo: all_to_all_single dispatch and
    combine between real processes."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_04667_b200 as fd
        from paper_2506_04667_b200.bulksync import BulkSyncMoE
        cfg = fd.MoeConfig(tokens_per_device=128, embed_dim=64, ffn_dim=96, experts_total=8, devices=world,
                           topk=2, seed=3)
        model = fd.make_model(cfg)
        shard = fd.make_shards(cfg)[rank]
        m = BulkSyncMoE(cfg, model, rank=rank, world=world, device="cpu")
        q.put((rank, m.forward(torch.from_numpy(shard)).numpy()))
    finally:
        dist.destroy_process_group()
