"""Certified-gate check at a headline shape: exact-fallback fraction, routing parity vs the oracle,
and gate-phase time in certified vs exact mode (device trace)."""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
from oracle import pyoracle as po
S = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
E = int(sys.argv[2]) if len(sys.argv) > 2 else 128
k = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=2048, ffn_dim=2048, experts_total=E, devices=1, topk=k)
model = fd.make_model(cfg)
shards = fd.make_shards(cfg)
op = fd.Operator(cfg); op.set_weights(model)
cap = fd.expert_capacity(cfg)
want = po.gate(shards[0], model.wg, k, cap)
for exact in (False, True):
    o = fd.ForwardOptions(exact_gate=exact)
    for _ in range(2):
        res = op.forward(shards, opts=o)
    g = res.gates[0]
    t = op.trace(0) / 1e3
    ok = (np.array_equal(g.picks_expert, want["picks_expert"]) and np.array_equal(g.picks_slot, want["picks_slot"])
          and np.array_equal(g.table_token, want["table_token"][:, :cap]) and g.dropped == want["dropped"])
    gerr = np.max(np.abs(g.g_phi.astype(np.float64) - want["g_phi"]) / np.maximum(np.abs(want["g_phi"]), 1e-30))
    print(f"exact_gate={exact}: routing_exact={ok} exact_tokens={res.stats[0].gate_exact_tokens}/{S} pair_tokens={res.stats[0].gate_pair_tokens} "
          f"gphi_maxrel={gerr:.2e} kernel_ms={res.stats[0].kernel_ms:.3f} gate_phase_us(med)={np.median(t[:, 1]-t[:, 0]):.1f}")
