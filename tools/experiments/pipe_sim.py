"""Toy discrete-time model of one SMSP + the tensor pipe of k_paged_attn_2cta, to compare
softmax/MMA orderings. Not a measurement: a planning aid (numbers in cycles, per 128-key page)."""
import sys

XU_PER_WARP = 384     # 48 MUFU x 8 cycles per warp per page-half (64 columns)
PRE = 250             # tmem load + (max) before the exponentials
TAIL = 150            # tmem st, fences, arrive
LAT = 120             # mbarrier / commit latencies MMA<->softmax


def sim(design, pages=200, s_cost=512, pv_cost=512):
    # tensor pipe: FIFO of (ready_time_of_issue, duration, name)
    t = 0
    tensor_free = 0
    s_done = {}          # (page, half) -> time S half available
    p_done = {}          # (page, half) -> time P ready
    pv_issued = {}
    # warps: state machine
    warps = [dict(w=0, page=0, phase="wait", rem=0, t_start=0), dict(w=1, page=0, phase="wait", rem=0, t_start=0)]
    if design == "stagger":
        warps[1]["page"] = 0
    # MMA issue plan: list of ops in order; each op has deps
    ops = []
    if design in ("base", "stagger"):
        ops += [("S", 0, None), ("S", 1, None)]
        for n in range(pages):
            ops += [("PV", n, 0), ("PV", n, 1), ("S", n + 2, None)]
    else:  # split
        ops += [("S", 0, 0), ("S", 0, 1), ("S", 1, 0), ("S", 1, 1)]
        for n in range(pages):
            ops += [("PV", n, 0), ("S", n + 2, 0), ("PV", n, 1), ("S", n + 2, 1)]
    oi = 0
    finish = {}
    xu_busy = 0
    end_page = {0: {}, 1: {}}
    while t < 400000:
        # MMA warp: issue next op if deps satisfied (issue latency folded into LAT)
        while oi < len(ops):
            kind, n, h = ops[oi]
            if kind == "PV":
                if p_done.get((n, h), 1e18) + LAT > t:
                    break
                start = max(t, tensor_free)
                tensor_free = start + pv_cost // 2
                pv_issued[(n, h)] = tensor_free
            else:
                if n >= pages:
                    oi += 1
                    continue
                dur = s_cost if h is None else int(s_cost / 2 / 0.8)
                start = max(t, tensor_free)
                tensor_free = start + dur
                for hh in ((0, 1) if h is None else (h,)):
                    s_done[(n, hh)] = tensor_free + LAT
            oi += 1
        # softmax warps
        in_xu = [w for w in warps if w["phase"] == "exp"]
        for w in warps:
            if w["page"] >= pages:
                continue
            n, h = w["page"], w["w"]
            if w["phase"] == "wait":
                if s_done.get((n, h), 1e18) <= t:
                    w["phase"], w["rem"] = "pre", PRE
            elif w["phase"] == "pre":
                w["rem"] -= 1
                if w["rem"] <= 0:
                    w["phase"], w["rem"] = "exp", XU_PER_WARP
            elif w["phase"] == "exp":
                w["rem"] -= 1.0 / len(in_xu)   # XU shared
                if w["rem"] <= 0:
                    w["phase"], w["rem"] = "tail", TAIL
            elif w["phase"] == "tail":
                w["rem"] -= 1
                if w["rem"] <= 0:
                    p_done[(n, h)] = t
                    end_page[h][n] = t
                    w["page"] += 1
                    w["phase"] = "wait"
        if all(w["page"] >= pages for w in warps) and oi >= len(ops):
            break
        t += 1
    per = (end_page[1][pages - 1] - end_page[1][pages // 2]) / (pages - 1 - pages // 2)
    return per


for d in ("base", "split"):
    print(d, round(sim(d), 1), "cycles/page")
