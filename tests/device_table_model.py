"""Python statement of the device balancer's rule (csrc/host_table.cpp):
the kernel routing of plan subtasks and the stream-K cut of tensor-core
work into per-CTA-pair pieces. tests/test_device_table.py checks the
library's task tables against it, record for record.

The rule ("Device balancer"): every tensor-core (TC) group is
(plan subtask, chunk of <= 256/g requests); a unit = (TC group, kv head) of
ceil(max_visible / 128) KV tiles. Units are laid out in lanes (lane c = the
c-th row chunk of every KV slice, then heads). With P CTA pairs, every pair gets T = ceil(W / P) tiles: lane c runs
on floor(W_c / T) pairs of its own -- pair k of a lane takes tiles
[k T, (k + 1) T) of the lane's unit sequence -- and the lane tails (what
does not fill a whole pair) are pooled in lane order and cut into T-tile
pieces for the remaining pairs. Pieces never cross units. Slices are
taken in order of decreasing lane count (then pool order), so every lane's
sequence is a prefix of lane 0's: pair k of every lane reads the same K/V
tiles at the same time."""
from __future__ import annotations

MULTI_ROWS, MULTI_MAX_ROWS, TC_MIN_ROWS, TC_ROWS = 32, 16, 16, 256
TCT_ROWS, TCT_MAX_ROWS = 128, 64


def route(n_live: int, g: int, multi: bool = True, force_tc: bool = False, node_rows: int = 0,
          tct: bool = True) -> str:
    rows = n_live * g
    lo = MULTI_MAX_ROWS + 1 if multi else TC_MIN_ROWS
    if tct and not force_tc and n_live >= 2 and node_rows <= TCT_MAX_ROWS:
        return "tct"
    if force_tc or rows >= lo:
        return "tc"
    if multi and n_live >= 2:
        return "multi"
    return "gemv"


def groups_of(forest, plan, g, multi=True, force_tc=False, tct=True):
    """[(kind, kv_tok, len, [(req, vis_local)], order)] in plan order, like
    the table builder (query-set chunks per task, rows with visible > start)."""
    qsets = {}
    for t_i, t in enumerate(plan.tasks):
        qsets.setdefault(t.node, []).append(t_i)
    chunk = {}
    for node, tis in qsets.items():
        qs = list(forest.node(node).query_set)
        tot = sum(plan.tasks[i].n_q for i in tis)
        hm = tot // len(qs)
        cur = 0
        for i in tis:
            k = plan.tasks[i].n_q // hm
            chunk[i] = qs[cur:cur + k]
            cur += k
    out = []
    for st in plan.subtasks:
        live = [(r, min(forest.visible_count(st.node, r), st.stop) - st.start) for r in chunk[st.task_index]
                if forest.visible_count(st.node, r) > st.start]
        if not live:
            continue
        kind = route(len(live), g, multi, force_tc, len(forest.node(st.node).query_set) * g, tct)
        per = {"tc": max(1, TC_ROWS // g), "tct": max(1, TCT_ROWS // g), "multi": max(1, MULTI_ROWS // g),
               "gemv": 1}[kind]
        for a in range(0, len(live), per):
            out.append((kind, forest.token_offset[st.node] + st.start, st.stop - st.start, live[a:a + per],
                        len(out)))
    return out


def tc_pieces(forest, plan, g, h_local, sms=148, budget=0, multi=True, force_tc=False, tct=True):
    """The TC piece records (kv_tok, len, n_rows, max_vis, qreq0, pair,
    head) in the table's order (pairs ascending), and the pair count."""
    groups = groups_of(forest, plan, g, multi, force_tc, tct)
    order = {"tc": 0, "gemv": 1, "multi": 3, "tct": 4}
    # kind, then longest slices first (stable)
    groups = sorted(groups, key=lambda x: (order[x[0]], -x[2]))
    tcg = [x for x in groups if x[0] == "tc"]
    if not tcg:
        return [], 0
    pairs = max(1, (min(sms, budget) if budget > 0 else sms) // 2)
    tiles = lambda x: (max(v for _, v in x[3]) + 127) // 128
    by_slice = {}
    for x in tcg:
        by_slice.setdefault((x[1], x[2]), []).append(x)
    lanes = []
    # slices with more lanes first (stable over pool order): the lanes'
    # sequences are prefixes of lane 0's, aligned position for position
    for key in sorted(sorted(by_slice), key=lambda k: -len(by_slice[k])):
        for c, x in enumerate(sorted(by_slice[key], key=lambda y: y[4])):
            if len(lanes) <= c:
                lanes.append([])
            lanes[c].append(x)
    lane_w = [sum(tiles(x) * h_local for x in lane) for lane in lanes]
    T = max(1, -(-sum(lane_w) // pairs))
    lane_p = [w // T for w in lane_w]
    used = sum(lane_p)
    pieces = []
    tail_pair, tail_pos, pair0 = used, 0, 0
    for c, lane in enumerate(lanes):
        if lane_w[c] == 0:
            continue
        main_end = lane_p[c] * T
        pos = 0
        for x in lane:
            nt = tiles(x)
            for h in range(h_local):
                t = 0
                while t < nt:
                    if pos < main_end:
                        k = pos // T
                        take = min(nt - t, (k + 1) * T - pos)
                        pair = pair0 + k
                    else:
                        k = tail_pos // T
                        take = min(nt - t, (k + 1) * T - tail_pos)
                        pair = tail_pair + min(k, max(0, pairs - 1 - tail_pair))
                        tail_pos += take
                    pieces.append((x, h, t, t + take, pair))
                    t += take
                    pos += take
        pair0 += lane_p[c]
    n_pairs = min(pairs, used + -(-tail_pos // T))
    recs = []
    for x, h, t0, t1, pair in pieces:
        tok0, tok1 = t0 * 128, min(t1 * 128, x[2])
        rows = [(r, min(v, tok1) - tok0) for r, v in x[3] if min(v, tok1) - tok0 > 0]
        if not rows:
            continue
        reqs = [r for r, _ in rows]
        q0 = reqs[0] if reqs == list(range(reqs[0], reqs[0] + len(reqs))) else -1
        recs.append((x[1] + tok0, tok1 - tok0, len(rows), max(v for _, v in rows), q0, pair, h))
    recs.sort(key=lambda r: r[5])  # stable: pairs ascending
    return recs, n_pairs
