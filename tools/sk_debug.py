"""Debug the forced stream-K path on a small shape: NaN rows, workspace fill sensitivity."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2605_16839_b200 as cpa
from synth.workload import random_qkv
from tests.gpu_helpers import Case
B, Hq, Hkv, bs, C, P = [int(x) for x in (sys.argv[1:] or "1 4 1 64 300 640".split())]
q, k, v = random_qkv(B, Hq, Hkv, 128, C, P + C, seed=B * 11 + C + bs)
ref = O.dense_causal_attention(q, k, v, P)
for fill in (0.0, float("nan")):
    for fl in (cpa.F_PERSIST, cpa.F_NO_PERSIST):
        case = Case(q, k, v, P, bs, seed=3, flags=cpa.F_OUT_F32 | fl)
        ws = torch.full((cpa.workspace_bytes(case.params) // 4,), fill, dtype=torch.float32, device="cuda")
        o = case.out(True)
        cpa.paged_attention(case.params, case.dq, case.cache, None, o, workspace=ws.view(torch.uint8))
        torch.cuda.synchronize()
        g = o.cpu().numpy().astype(np.float64)
        bad = np.argwhere(~np.isfinite(g).all(axis=-1))
        err = np.nanmax(np.abs(g - ref)) / np.sqrt(np.mean(ref ** 2))
        print(f"fill={fill} flags={fl}: nonfinite rows {len(bad)} first {bad[:6].tolist()} maxerr {err:.3e}")
        if len(bad):
            ps = sorted(set(int(x[1]) for x in bad))
            print("   bad positions p:", ps[:20], "...", ps[-5:], "heads", sorted(set(int(x[2]) for x in bad)))
# detail for the forced stream-K run
case = Case(q, k, v, P, bs, seed=3, flags=cpa.F_OUT_F32 | cpa.F_PERSIST)
ws = torch.zeros(cpa.workspace_bytes(case.params), dtype=torch.uint8, device="cuda")
o = case.out(True)
cpa.paged_attention(case.params, case.dq, case.cache, None, o, workspace=ws)
torch.cuda.synchronize()
g = o.cpu().numpy()
nqt = -(-C // 128)
U = nqt * B * (Hq // (Hq // Hkv)) * ((Hq // Hkv) // 2)
wsi = ws.view(torch.int32).cpu().numpy()
stride = ((U + 1) * 4 + 255) // 256 * 64
pre, ln, st, nd = (wsi[i * stride:i * stride + U + 1] for i in range(4))
print("U", U, "pre", pre.tolist(), "len", ln[:U].tolist(), "start", st[:U].tolist(), "nd", nd[:U].tolist())
for qt in range(nqt):
    for h in range(Hq):
        blk = g[0, qt * 128:(qt + 1) * 128, h]
        nn, ni = int(np.isnan(blk).any(axis=-1).sum()), int(np.isinf(blk).any(axis=-1).sum())
        if nn or ni:
            rows = np.where(~np.isfinite(blk).all(axis=-1))[0]
            print(f"qt {qt} h {h}: nan rows {nn} inf rows {ni} rows {rows.min()}..{rows.max()}")
# partial slot of cluster 63 (share [69,70) = u4's page t=11 at this shape)
wsf = ws.view(torch.float32).cpu().numpy()
up = lambda x: (x + 255) // 256 * 256
off_o = 4 * up((U + 1) * 4)
nslots = 80 * (B * Hq // (Hq // Hkv)) * 2
off_ml = off_o + up(nslots * 256 * 128 * 4)
for c in (63, 62, 39):
    slot = c * 2
    po = wsf[(off_o // 4) + slot * 256 * 128:(off_o // 4) + (slot + 1) * 256 * 128].reshape(256, 128)
    pm = wsf[(off_ml // 4) + slot * 512:(off_ml // 4) + (slot + 1) * 512].reshape(256, 2)
    print(f"cluster {c} slot0: O nan rows {int(np.isnan(po).any(1).sum())} inf rows {int(np.isinf(po).any(1).sum())}; "
          f"m[0:3] {pm[:3, 0].tolist()} l[0:3] {pm[:3, 1].tolist()} m[100] {pm[100].tolist()} O[0,:4] {po[0, :4].tolist()}")
