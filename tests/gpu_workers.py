"""Subprocess bodies for the GPU tests that need their own process:

* ``ipc``: one rank of a two-process expert-parallel forward on ONE B200. Each process owns one rank
  (its own CUDA context); the symmetric heaps are cross-mapped with CUDA IPC handles exchanged over
  torch.distributed (gloo), exactly as under torchrun on 8 GPUs (dist.attach_peers). The kernels then
  exchange dispatch rows, combine rows and epoch flags through the IPC mappings: the multi-process data
  path (fdmoe_runtime.cpp fdmoe_export_heap / fdmoe_import_peers; runtime.hpp:332-372, 667-699,
  pgas.hpp:99-122). Without MPS the two contexts time-slice the GPU, so every cross-process wait spans a
  scheduler time slice: correctness, not speed, is what this exercises.
* ``fault``: the development library with FDMOE_DEBUG fault injection (over-subscribed packet ->
  ProtocolError, pgas.hpp:101-112), then a clean forward on the same operator (recovery).

Usage: python tests/gpu_workers.py ipc RANK WORLD PORT PREC OUT.npz
       python tests/gpu_workers.py fault OUT.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def ipc_cfg(fd, world, prec):
    return fd.MoeConfig(tokens_per_device=384, embed_dim=256, ffn_dim=512, experts_total=8, devices=world, topk=2,
                        precision=prec, seed=21)


def run_ipc(rank, world, port, prec, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_04667_b200 as fd
        from paper_2506_04667_b200 import dist as fdist
        cfg = ipc_cfg(fd, world, prec)
        op = fd.Operator(cfg, device_ids=[0], first_rank=rank, n_local=1)
        fdist.attach_peers(op)
        op.set_weights(fd.make_model(cfg))
        shard = fd.make_shards(cfg)[rank]
        opts = fd.ForwardOptions(deadlock_budget_ms=120000)
        outs, tabs, stats = [], [], []
        for mode in (fd.ScheduleMode.overlapped, fd.ScheduleMode.overlapped, fd.ScheduleMode.sequential):
            opts.mode = mode
            dist.barrier()
            r = op.forward([shard], opts)
            outs.append(r.outputs[0])
            tabs.append(r.gates[0].table_token)
            s = r.stats[0]
            stats.append([s.gemm0, s.gemm1, s.combine, s.executed, s.bound_final, s.scheduled_final])
        info = op.info()
        op.close()
        np.savez(out, outs=np.stack(outs), tabs=np.stack(tabs), stats=np.array(stats, np.int64),
                 fused=np.int64(info["fused_combine"]))
    finally:
        dist.destroy_process_group()


def run_fault(out):
    import paper_2506_04667_b200 as fd
    fd.select_library(fd._build.DEV_LIB)
    cfg = fd.MoeConfig(tokens_per_device=256, embed_dim=128, ffn_dim=256, experts_total=8, devices=2, topk=2,
                       seed=5)
    model = fd.make_model(cfg)
    shards = fd.make_shards(cfg)
    op = fd.Operator(cfg)
    op.set_weights(model)
    res = {}
    os.environ["FDMOE_DEBUG"] = "8192"   # kDbgInjectOversub
    try:
        op.forward(shards, fd.ForwardOptions(deadlock_budget_ms=2000))
        res["first"] = "no error"
    except fd.ProtocolError as e:
        res["first"] = "ProtocolError: " + str(e)
    except Exception as e:  # noqa: BLE001
        res["first"] = type(e).__name__ + ": " + str(e)
    del os.environ["FDMOE_DEBUG"]
    r = op.forward(shards)
    res["outputs"] = [o.tolist() for o in r.outputs]
    op.close()
    json.dump(res, open(out, "w"))


if __name__ == "__main__":
    if sys.argv[1] == "ipc":
        run_ipc(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6])
    elif sys.argv[1] == "fault":
        run_fault(sys.argv[2])
    else:
        raise SystemExit("unknown worker " + sys.argv[1])
