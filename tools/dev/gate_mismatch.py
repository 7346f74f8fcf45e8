"""Which tokens does the tensor-core gate route differently from the oracle, and where do they sit
(position inside their CTA's token range = which 128-token gate tile)?"""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
from oracle import pyoracle as po

S, E, P = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = fd.MoeConfig(tokens_per_device=S, embed_dim=2048, ffn_dim=2048, experts_total=E, devices=P, topk=2, seed=0)
model = fd.make_model(cfg)
shards = fd.make_shards(cfg)
op = fd.Operator(cfg, device_ids=[0] * P)
op.set_weights(model)
res = op.forward(shards)
cpr = op.info()["ctas_per_rank"]
nblk = (S + 15) // 16
for d in range(P):
    cap = fd.expert_capacity(cfg)
    want = po.gate(shards[d], model.wg, 2, cap)
    g = res.gates[d]
    bad = np.nonzero(np.any(g.picks_expert != want["picks_expert"], axis=1))[0]
    print(f"rank {d}: {bad.size} tokens with different picks")
    for t in bad[:10]:
        blk = t // 16
        cta = next(c for c in range(cpr) if nblk * c // cpr <= blk < nblk * (c + 1) // cpr)
        tokA = nblk * cta // cpr * 16
        z = np.zeros(E, np.float32)
        a = shards[d][t]
        for x in range(2048):
            z = (z + (a[x] * model.wg[x]).astype(np.float32)).astype(np.float32)
        top = np.argsort(-z)[:4]
        print(f"  tok {t} cta {cta} pos {t - tokA} ours {g.picks_expert[t]} ref {want['picks_expert'][t]} "
              f"top4 {top} z {z[top]} gaps {np.diff(z[top])}")
op.close()

# where did the wrong rows come from? match our G_phi (log) against every token's reference logits
print("--- provenance of wrong rows (rank 0) ---")
op = fd.Operator(cfg, device_ids=[0] * P)
op.set_weights(model)
res = op.forward(shards)
want = po.gate(shards[0], model.wg, 2, fd.expert_capacity(cfg))
g = res.gates[0]
bad = np.nonzero(np.any(g.picks_expert != want["picks_expert"], axis=1))[0]
zall = shards[0].astype(np.float64) @ model.wg.astype(np.float64)
for t in bad[:6]:
    lg = np.log(np.maximum(g.g_phi[t].astype(np.float64), 1e-30))
    lg -= lg.mean()
    zc = zall - zall.mean(1, keepdims=True)
    d = np.abs(zc - lg[None, :]).max(1)
    best = np.argsort(d)[:3]
    print(f"tok {t}: best matching token rows {best} (max dev {d[best]}) own dev {d[t]:.3e}")
op.close()

print("--- which 64-K chunk is off? (rank 0) ---")
a0 = shards[0].astype(np.float64)
W = model.wg.astype(np.float64)
for t in bad[:6]:
    lg = np.log(np.maximum(g.g_phi[t].astype(np.float64), 1e-30))
    chunks = np.stack([a0[t, j * 64:(j + 1) * 64] @ W[j * 64:(j + 1) * 64] for j in range(32)])  # 32 x E
    delta = lg - zall[t]
    delta -= delta.mean()
    best = []
    for j in range(32):
        for sgn in (1, -1):
            c = sgn * chunks[j]
            r = delta - (c - c.mean())
            best.append((np.abs(r).max(), j, sgn))
    for i2 in range(32):
        for j2 in range(32):
            if i2 != j2:
                c = chunks[i2] - chunks[j2]
                r = delta - (c - c.mean())
                best.append((np.abs(r).max(), (i2, j2), 0))
    best.sort(key=lambda x: x[0])
    print(f"tok {t}: |delta| {np.abs(delta).max():.3f}; best explanations {best[:3]}")

print("--- chunk provenance vs tile-1 token (tok-128) ---")
for t in bad[:8]:
    lg = np.log(np.maximum(g.g_phi[t].astype(np.float64), 1e-30))
    delta = lg - zall[t]; delta -= delta.mean()
    best = []
    for src in (t - 128, t - 64, t + 128 - 256):
        for half in range(64):   # 32-K half stages
            c = a0[src, half * 32:(half + 1) * 32] @ W[half * 32:(half + 1) * 32] - a0[t, half * 32:(half + 1) * 32] @ W[half * 32:(half + 1) * 32]
            r = delta - (c - c.mean())
            best.append((round(float(np.abs(r).max()), 4), src - t, half))
    best.sort()
    print(f"tok {t}: |delta| {np.abs(delta).max():.3f} best {best[:3]}")

print("--- stale-ring explanations ---")
for t in bad[:8]:
    lg = np.log(np.maximum(g.g_phi[t].astype(np.float64), 1e-30))
    delta = lg - zall[t]; delta -= delta.mean()
    best = []
    A = a0[t]
    for kb in range(32):
        ks = slice(kb * 64, (kb + 1) * 64)
        base = A[ks] @ W[ks]
        for d2 in (-4, -2, -1, 1, 2, 4):
            kb2 = kb + d2
            if not 0 <= kb2 < 32:
                continue
            ks2 = slice(kb2 * 64, (kb2 + 1) * 64)
            cB = A[ks] @ W[ks2] - base          # stale Wg (B) stage
            cA = A[ks2] @ W[ks] - base          # stale token (A) data
            for name, c in (("B", cB), ("A", cA)):
                r = delta - (c - c.mean())
                best.append((round(float(np.abs(r).max()), 4), name, kb, d2))
        for half in range(2):
            hs = slice(kb * 64 + half * 32, kb * 64 + half * 32 + 32)
            c = -(A[hs] @ W[hs])                # a lost half-stage
            r = delta - (c - c.mean()); best.append((round(float(np.abs(r).max()), 4), "lost-half", kb, half))
            r = delta + (c - c.mean()); best.append((round(float(np.abs(r).max()), 4), "double-half", kb, half))
    best.sort()
    print(f"tok {t}: |delta| {np.abs(delta).max():.3f} best {best[:3]}")
