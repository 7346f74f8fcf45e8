"""Bulk-synchronous expert-parallel MoE layer: separate kernels + NCCL all-to-all.

This is the comparison the paper's overlap efficiency is defined against: the
reference's ScheduleMode::sequential (runtime.hpp:175-198, 885-908) rebuilt the way a conventional GPU
MoE layer runs it -- every stage a separate library kernel, and the token exchange a bulk-synchronous
NCCL all-to-all between them:

    gate GEMM -> softmax -> top-k -> capacity slots      (gate.hpp:57-106)
    pack per (destination, local expert, slot)            (runtime.hpp:332-372, padded to C rows)
    NCCL all_to_all_single                                (dispatch)
    expert FFN as batched cuBLAS GEMMs (+bias, act)       (runtime.hpp:652-699)
    NCCL all_to_all_single                                (combine return)
    weighted scatter-add into token order                 (runtime.hpp:701-712)

FP32 throughout (cuBLAS SGEMM, TF32 disabled) so it computes the same FP32 layer as the fused
kernel's FP32-accurate mode. It is a baseline, not a product path: the fused single launch
(`Operator.forward_device`) is what bench.py's `value` measures. Ties in top-k follow torch.topk, so
routing may differ from the reference on exact logit ties (absent in the seeded workloads).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class BulkSyncMoE:
    """One rank's state: its local experts' weights and the gate, on `device`."""

    def __init__(self, cfg, model, rank: int = 0, world: int = 1, device="cuda"):
        self.cfg, self.rank, self.world = cfg, rank, world
        self.E = cfg.experts_total
        self.El = self.E // world
        self.H, self.D, self.k = cfg.embed_dim, cfg.ffn_dim, cfg.topk
        S = cfg.tokens_per_device
        q = cfg.capacity_factor * S / self.E   # config.hpp:89-100
        self.C = max(1, int(-(-(q - 1e-9) // 1)))
        lo, hi = rank * self.El, (rank + 1) * self.El
        t = lambda a: torch.as_tensor(a).to(device=device, dtype=torch.float32).contiguous()  # noqa: E731
        self.wg = t(model.wg)
        self.w1, self.b1 = t(model.w1[lo:hi]), t(model.b1[lo:hi]).unsqueeze(1)
        self.w2, self.b2 = t(model.w2[lo:hi]), t(model.b2[lo:hi]).unsqueeze(1)
        self.act = {0: torch.relu, 1: torch.nn.functional.gelu, 2: lambda x: x}[getattr(cfg, "activation", 0)]
        self.send = torch.empty(world * self.El * self.C, self.H, device=device)
        self.recv = torch.empty_like(self.send)

    def _a2a(self, out, inp):
        if self.world > 1:
            dist.all_to_all_single(out, inp)
        else:
            out.copy_(inp)   # one rank: the exchange is a local copy (still a separate kernel)

    @torch.no_grad()
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            return self._forward(x)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev

    def _forward(self, x):
        S, H, E, C, k = x.shape[0], self.H, self.E, self.C, self.k
        # gate: logits, softmax, top-k, normalised weights (gate.hpp:57-95)
        p = torch.softmax(x @ self.wg, dim=1)
        pv, pe = torch.topk(p, k, dim=1)
        w = pv / pv.sum(dim=1, keepdim=True)
        # capacity: slot = rank of the token among those that picked the expert, by token id (gate.hpp:94-103)
        onehot = torch.zeros(S, E, dtype=torch.int32, device=x.device)
        onehot.scatter_(1, pe, 1)
        pos = torch.cumsum(onehot, dim=0) - 1
        slot = torch.gather(pos, 1, pe)                          # S x k
        keep = slot < C
        tok = torch.arange(S, device=x.device).unsqueeze(1).expand(S, k)[keep]
        dst = (pe * C + slot)[keep]                              # row in the [E, C] send layout
        wk = w[keep]
        # pack (padding rows stay zero) and dispatch
        self.send.zero_()
        self.send.index_copy_(0, dst, x.index_select(0, tok))
        self._a2a(self.recv, self.send)
        # expert FFN: recv is [src, El, C, H] -> [El, src*C, H]
        xe = self.recv.view(self.world, self.El, C, H).transpose(0, 1).reshape(self.El, self.world * C, H)
        h = self.act(torch.baddbmm(self.b1, xe, self.w1))
        y = torch.baddbmm(self.b2, h, self.w2)
        self.send.view(self.world, self.El, C, H).copy_(y.view(self.El, self.world, C, H).transpose(0, 1))
        self._a2a(self.recv, self.send)                          # combine return: rows back to the origin
        out = torch.zeros(S, H, device=x.device)
        out.index_add_(0, tok, self.recv.index_select(0, dst) * wk.unsqueeze(1))
        return out
