"""Pipeline skeleton (148 CTAs): converged single issuer warp (2048) vs two issuer warps alternating half-stages
with a named-barrier hand-off (4096), with the A-ring handshake (2), converter tcgen05.st (4) and the token
ring (8); 1024 = valid A data; 1 = corr/main accumulators."""
import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2506_04667_b200 as fd
for base, n in ((1, "corr/main free-running"), (3, "+ A-ring handshake"), (7, "+ converter tcgen05.st"),
                (15, "+ token-ring handshake")):
    out = []
    for extra in (2048, 4096):
        v = C.c_double()
        fd.dev_check(fd.dev_lib().fdmoe_debug_mma_rate(16 + (base | extra | 1024), 1, 128, 4000, C.byref(v)))
        out.append(v.value)
    print(f"{n:28s}: one converged issuer {out[0]:6.1f}   ping-pong issuers {out[1]:6.1f} cyc/mma", flush=True)
