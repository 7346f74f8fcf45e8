import sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
from oracle import pyoracle as po
for P in (1, 2):
    cfg = fd.MoeConfig(tokens_per_device=256, embed_dim=128, ffn_dim=256, experts_total=8, devices=P, topk=2, seed=5)
    model = fd.make_model(cfg)
    op = fd.Operator(cfg); op.set_weights(model)
    for it in range(4):
        shards = fd.make_shards(cfg, seed=100 + (it // 2))
        res = op.forward(shards)
        for d in range(P):
            want = po.dense_forward(shards[d], model, cfg, threads=8)
            got = res.outputs[d]
            err = np.abs(got - want).max(axis=1)
            bad = np.nonzero(err > 1e-4)[0]
            print(f"P={P} it={it} rank={d} rel={fd.max_rel_error([got],[want]):.2e} badrows={bad.size} first={bad[:10]} stats={res.stats[d]}")
            if bad.size:
                t = bad[0]
                print("  picks", res.gates[d].picks_expert[t], res.gates[d].picks_slot[t], "got[:4]", got[t,:4], "want[:4]", want[t,:4])
    op.close()
