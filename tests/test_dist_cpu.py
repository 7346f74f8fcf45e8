"""Multi-process host logic (world_size 2, gloo on CPU): heap-blob exchange, max-over-ranks timing,
and the reference's bytes matrix assembled from per-rank routing — what bench.py / a torchrun
deployment run before and after the (GPU-only) layer launch."""
import multiprocessing as mp
import socket

import numpy as np

import paper_2506_04667_b200 as fd
from oracle import pyoracle as po


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_bootstrap_gloo():
    import dist_workers
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=dist_workers.run, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_blobs = [bytes([r]) * 64 + b"heap" for r in range(world)]
    cfg = fd.MoeConfig(tokens_per_device=256, embed_dim=64, ffn_dim=64, experts_total=8, devices=world, topk=2,
                       seed=4)
    model = fd.make_model(cfg)
    counts = [po.gate(s, model.wg, 2, fd.expert_capacity(cfg))["slot_counts"] for s in fd.make_shards(cfg)]
    want_payload = fd.payload_bytes(cfg, counts)
    for r in range(world):
        assert got[r]["blobs"] == want_blobs
        assert got[r]["max"] == 1.25
        assert np.array_equal(got[r]["payload"], want_payload)
        assert got[r]["experts"] == list(range(r * 4, r * 4 + 4))
