"""Generate golden fixtures from the REFERENCE ITSELF (oracle/_ref/libmoefabric_ref.so,
built from /root/reference by oracle/Makefile). Run in the dev container:

    make -C oracle && python tests/golden/make_golden.py

Each fixture stores the config, the reference dense_moe_forward() outputs, forward()'s outputs and routing tables
(T_phi, G_phi, slot counts) per device, and a prefix of the seeded inputs so the input
generator (harness.hpp:76-109 restated in libfdmoe) is pinned as well.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2506_04667_b200 as fd  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

FIXTURES = {
    # name: (S, H, D, E, P, k, cf, act, seed)
    "mini_p1": (64, 64, 64, 8, 1, 2, 1.0, 0, 0),
    "mini_p2": (64, 64, 96, 8, 2, 2, 1.0, 0, 1),
    "mini_p4_gelu": (48, 32, 64, 8, 4, 2, 1.5, 1, 2),
    "mini_k3": (40, 32, 32, 6, 1, 3, 0.75, 2, 3),
    "c1_shape_small": (128, 128, 256, 8, 1, 2, 1.0, 0, 0),
}


def main():
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name, (S, H, D, E, P, k, cf, act, seed) in FIXTURES.items():
        cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=H, ffn_dim=D, experts_total=E, devices=P, topk=k,
                           capacity_factor=cf, activation=act, tile_rows=16, tile_cols=8, seed=seed)
        model = fd.make_model(cfg)
        shards = fd.make_shards(cfg)
        rm = po.RefModel(model, cfg)
        r = po.ref_forward(cfg, shards, rm, processors=4)
        # dense_moe_forward (oracle.hpp:116) is the deterministic reference output; the runtime's
        # forward() equals it bit for bit for k <= 2 and to rounding for k >= 3 (its combine adds
        # arrive in task order, runtime.hpp:701-712)
        dense = np.stack([po.ref_dense_forward(cfg, shards[d], rm) for d in range(P)])
        np.savez_compressed(
            os.path.join(out_dir, name + ".npz"),
            meta=np.array([S, H, D, E, P, k, act, seed], np.int64), cf=np.float64(cf),
            outputs=dense, forward_outputs=r["outputs"], table_token=r["table_token"], table_weight=r["table_weight"],
            slot_counts=r["slot_counts"], g_phi=r["g_phi"], bytes=r["bytes"],
            shard_head=np.stack(shards).view(np.uint32)[..., :4].ravel()[:64])
        print("wrote", name)


if __name__ == "__main__":
    main()
