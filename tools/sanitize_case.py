"""Small chunk steps for compute-sanitizer (memcheck / racecheck / synccheck): the tiny config (d=64,
bs=16: 1-CTA kernel), a 2-CTA config (d=128, bs=128, with a partial last q-tile), the fp16 V pool, the
persistent stream-K grid, the exact scorer and MASK_IN tables. Exits non-zero on a wrong result.

  compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_16839_b200 as cpa
from synth.workload import page_layout, random_qkv, to_pool


def case(Hq, Hkv, d, bs, C, P, flags=0, vf16=False):
    q, k, v = random_qkv(1, Hq, Hkv, d, C, P + C, seed=d + bs + C)
    L = P + C
    pt, npg = page_layout(1, -(-L // bs), 3)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)
    vp = dev(to_pool(v, pt, npg, bs))
    if vf16:
        vp = vp.half()
        flags |= cpa.F_V_F16
    cache = cpa.PagedKVCache(dev(to_pool(k, pt, npg, bs)), vp, torch.from_numpy(pt).cuda())
    p = cpa.make_params(1, Hq, Hkv, d, bs, C, P, alpha=0.06, flags=flags | cpa.F_OUT_F32)
    t = cpa.alloc_tables(p, mask=True)
    o = torch.empty(1, C, Hq, d, dtype=torch.float32, device="cuda")
    kc = dev(k[:, :, P:].transpose(0, 2, 1, 3))
    vc = dev(v[:, :, P:].transpose(0, 2, 1, 3))
    cpa.chunk_step(p, dev(q), cache, t, o, kc, vc)
    torch.cuda.synchronize()
    assert torch.isfinite(o).all()
    return o, t


if __name__ == "__main__":
    torch.cuda.set_device(0)
    case(8, 2, 64, 16, 64, 448)                                   # tiny: 1-CTA kernel
    case(8, 2, 128, 128, 200, 384)                                # 2-CTA pair, partial q-tile
    case(8, 2, 128, 128, 256, 512, vf16=True)                     # fp16 V pool
    case(8, 2, 128, 128, 256, 512, flags=cpa.F_PERSIST)           # persistent stream-K grid
    case(8, 2, 128, 64, 130, 256, flags=cpa.F_EXACT_SCORES)       # NEXT-1 exact scorer, bs 64
    o, t = case(8, 2, 128, 128, 256, 512, flags=cpa.F_MASK_OUT)
    p = cpa.make_params(1, 8, 2, 128, 128, 256, 512, flags=cpa.F_MASK_IN)
    cpa.build_tables(p, None, cpa.PagedKVCache(torch.zeros(1, 2, 128, 128, dtype=torch.bfloat16, device="cuda"),
                                               torch.zeros(1, 2, 128, 128, dtype=torch.bfloat16, device="cuda"),
                                               torch.zeros(1, 6, dtype=torch.int32, device="cuda")), t)
    torch.cuda.synchronize()
    print("sanitize cases ok")
