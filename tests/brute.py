"""Independent brute-force references used to PIN the oracle (tests only).

Nothing here calls oracle/ or the CUDA path.  Each routine computes a
quantity from its plain definition by exhaustive enumeration on tiny inputs:

* elmore_bruteforce: SPEC.md:434 -- Elmore(sink) = sum_k C_k * R(path(root,k)
  intersect path(root,sink)), the shared-path double loop.
* longest_path_levels: SPEC.md:257/267 -- level = length of the longest path
  from any source, by enumerating every path.
* path_enumeration_timing: SPEC.md:539/688 -- with frozen (slew-independent)
  delays, AT_L = max and AT_E = min over enumerated source->v paths with
  rise/fall tracking; RAT by enumerating v->endpoint paths.
"""
from __future__ import annotations

import math
from collections import defaultdict

import numpy as np

from synth.design import (NO_PIN, ROLE_FF_CK, SENSE_POS, SENSE_NEG, SENSE_NON,
                          SENSE_RISE_EDGE, SENSE_FALL_EDGE, Library)

INF = math.inf


def elmore_bruteforce(parent, R, C):
    """parent[i] (local, -1 root), R[i] edge parent->i, C[i] node cap (total)."""
    n = len(parent)

    def path_edges(i):
        e = set()
        while i > 0:
            e.add(i)
            i = parent[i]
        return e

    paths = [path_edges(i) for i in range(n)]
    out = []
    for s in range(n):
        tot = 0.0
        for k in range(n):
            shared = paths[s] & paths[k]
            tot += C[k] * sum(R[j] for j in shared)
        out.append(tot)
    return out


def _fanin_lists(d):
    """Explicit arc list: (u, v, kind, sense, tab) with kind 'net'/'cell'."""
    arcs = []
    for n in range(d.num_nets):
        b, e = int(d.net_ptr[n]), int(d.net_ptr[n + 1])
        drv = int(d.net_pins[b])
        for j in range(b + 1, e):
            arcs.append((drv, int(d.net_pins[j]), "net", SENSE_POS, None))
    for a in range(d.num_arcs):
        arcs.append((int(d.arc_from[a]), int(d.arc_to[a]), "cell", int(d.arc_sense[a]),
                     int(d.arc_tab[a])))
    return arcs


def longest_path_levels(d):
    arcs = _fanin_lists(d)
    succ = defaultdict(list)
    indeg = np.zeros(d.num_pins, int)
    for u, v, *_ in arcs:
        succ[u].append(v)
        indeg[v] += 1
    level = np.zeros(d.num_pins, int)

    def walk(u, length):      # enumerate every path
        if length > level[u]:
            level[u] = length
        for v in succ[u]:
            walk(v, length + 1)

    for s in range(d.num_pins):
        if indeg[s] == 0:
            walk(s, 0)
    return level


def _pairs(sense):
    return {SENSE_POS: [(0, 0), (1, 1)], SENSE_NEG: [(0, 1), (1, 0)],
            SENSE_NON: [(0, 0), (0, 1), (1, 0), (1, 1)],
            SENSE_RISE_EDGE: [(0, 0), (0, 1)], SENSE_FALL_EDGE: [(1, 0), (1, 1)]}[sense]


def const_value(lib: Library, t: int) -> float:
    _, _, v = lib.table(t)
    assert v.size == 1
    return float(v.reshape(-1)[0])


def path_enumeration_timing(d, elm_of_pin, off=None):
    """Frozen-delay brute force.  The library must hold 1x1 (constant) tables so
    that every arc delay is independent of slew and load.  elm_of_pin[p] is the
    net-arc delay into sink p (from elmore_bruteforce).  Returns at, rat,
    slack [P][4] (E_r, E_f, L_r, L_f) and res (WNS_s, TNS_s, WNS_h, TNS_h)."""
    lib = d.libs[0]
    cons = d.cons
    T = float(cons.period)
    arcs = _fanin_lists(d)
    if off is not None:                 # case analysis: disabled arcs (canonical order) left out
        arcs = [a for a, o in zip(arcs, off) if not o]
    P = d.num_pins
    succ = defaultdict(list)
    indeg = np.zeros(P, int)
    for (u, v, kind, sense, tab) in arcs:
        if kind == "net":
            dl = {(0, 0): elm_of_pin[v], (1, 1): elm_of_pin[v]}
        else:
            dl = {(i, o): max(0.0, const_value(lib, tab + o)) for (i, o) in _pairs(sense)}
        succ[u].append((v, dl))
        indeg[v] += 1

    # source arrival seeds
    seed_at = {}
    for k in range(cons.pi_pin.size):
        p = int(cons.pi_pin[k])
        if indeg[p] == 0:
            seed_at[p] = [float(x) for x in cons.pi_at[k]]
    for p in range(P):
        if int(d.pin_role[p]) == ROLE_FF_CK and indeg[p] == 0:
            seed_at[p] = [0.0, T / 2, 0.0, T / 2]

    at = np.empty((P, 4))
    at[:, 0:2] = INF
    at[:, 2:4] = -INF

    def fwd(v, orf, acc_e, acc_l):
        at[v, orf] = min(at[v, orf], acc_e)
        at[v, 2 + orf] = max(at[v, 2 + orf], acc_l)
        for (w, dl) in succ[v]:
            for (i, o), x in dl.items():
                if i == orf:
                    fwd(w, o, acc_e + x, acc_l + x)

    for s, a in seed_at.items():
        for rf in (0, 1):
            # early and late walk the same paths with the same frozen delays
            fwd(s, rf, a[rf], a[2 + rf])

    # endpoint seeds
    seed_l = defaultdict(lambda: [INF, INF])
    seed_e = defaultdict(lambda: [-INF, -INF])
    for k in range(cons.po_pin.size):
        p = int(cons.po_pin[k])
        for rf in (0, 1):
            seed_l[p][rf] = min(seed_l[p][rf], T - float(cons.po_out_max[k, rf]))
            seed_e[p][rf] = max(seed_e[p][rf], -float(cons.po_out_min[k, rf]))
    for c in range(d.num_checks):
        p, tb = int(d.chk_d[c]), int(d.chk_tab[c])
        for rf in (0, 1):
            if math.isfinite(at[p, 2 + rf]):
                seed_l[p][rf] = min(seed_l[p][rf], T - const_value(lib, tb + rf))
            if math.isfinite(at[p, rf]):
                seed_e[p][rf] = max(seed_e[p][rf], const_value(lib, tb + 2 + rf))
    endpoints = sorted(set(seed_l) | set(seed_e))

    rat = np.empty((P, 4))
    rat[:, 0:2] = -INF
    rat[:, 2:4] = INF

    def bwd(u, irf):
        """all (sum of delays, endpoint, orf) reachable from (u, irf)."""
        out = []

        def walk(v, rf, acc):
            if v in seed_l or v in seed_e:
                out.append((acc, v, rf))
            for (w, dl) in succ[v]:
                for (i, o), x in dl.items():
                    if i == rf:
                        walk(w, o, acc + x)
        walk(u, irf, 0.0)
        return out

    def bwd_strict(u, irf):
        """(sum, endpoint, orf) over paths with at least one arc."""
        out = []
        for (w, dl) in succ[u]:
            for (i, o), x in dl.items():
                if i == irf:
                    out.extend((acc + x, e, rf) for acc, e, rf in bwd(w, o))
        return out

    for u in range(P):
        for irf in (0, 1):
            # the pin's own seed (PO seeds are unconditional; D-pin seeds were
            # only created where the data arrival is defined) ...
            if u in seed_l:
                rat[u, 2 + irf] = seed_l[u][irf]
            if u in seed_e:
                rat[u, irf] = seed_e[u][irf]
            # ... and every path of length >= 1 to an endpoint, counted only
            # when the pin's arrival of that edge is defined
            reach = bwd_strict(u, irf)
            if math.isfinite(at[u, 2 + irf]):
                for acc, e, orf in reach:
                    rat[u, 2 + irf] = min(rat[u, 2 + irf], seed_l[e][orf] - acc)
            if math.isfinite(at[u, irf]):
                for acc, e, orf in reach:
                    rat[u, irf] = max(rat[u, irf], seed_e[e][orf] - acc)

    slack = np.full((P, 4), INF)
    for p in range(P):
        for rf in (0, 1):
            if math.isfinite(at[p, 2 + rf]) and math.isfinite(rat[p, 2 + rf]):
                slack[p, 2 + rf] = rat[p, 2 + rf] - at[p, 2 + rf]
            if math.isfinite(at[p, rf]) and math.isfinite(rat[p, rf]):
                slack[p, rf] = at[p, rf] - rat[p, rf]
    ws = [min(slack[e, 2], slack[e, 3]) for e in endpoints]
    wh = [min(slack[e, 0], slack[e, 1]) for e in endpoints]
    res = (min(ws, default=INF), sum(min(0.0, x) for x in ws),
           min(wh, default=INF), sum(min(0.0, x) for x in wh))
    return at, rat, slack, res


def constant_library_like(lib: Library, rng, lo=1.0, hi=10.0, chk=None) -> Library:
    """Replace every table of `lib` by a random 1x1 constant table."""
    tables = []
    for t in range(lib.num_tables):
        tables.append(([0.0], [0.0], [[float(np.round(rng.uniform(lo, hi), 3))]]))
    return Library.from_tables(tables)


def design_node_caps(d, corner=0):
    """Total node capacitance (wire + pin + PO load) per RC node, float64."""
    rc = d.rc[corner]
    po_ld = np.zeros(d.num_pins)
    for k in range(d.cons.po_pin.size):
        po_ld[int(d.cons.po_pin[k])] += float(d.cons.po_load[k])
    caps = rc.cap.astype(np.float64).copy()
    has = rc.node_pin != NO_PIN
    caps[has] += d.pin_cap[rc.node_pin[has]].astype(np.float64) + po_ld[rc.node_pin[has]]
    return caps


def path_list_bruteforce(d, elm_of_pin, mode="setup"):
    """Every timing path of a frozen-delay design by exhaustive DFS (SPEC.md
    path-report acceptance: "report_paths(k=inf) returns exactly the set of
    valid paths found by exhaustive DFS ... identical sort order"), as
    (slack, endpoint, ((pin, rf), ...) startpoint first, arrivals), sorted in
    report order: slack, endpoint id, then the (pin, rf) sequence read
    backwards from the endpoint.  Startpoints: pins without fan-in carrying a
    PI / ideal-clock arrival; endpoints: POs and checked D pins with a seed
    for that transition (PO: T - out_max / -out_min; check: T - setup /
    hold, defined where the data arrival of that edge is)."""
    lib = d.libs[0]
    cons = d.cons
    T = float(cons.period)
    late = mode == "setup"
    arcs = _fanin_lists(d)
    P = d.num_pins
    succ = defaultdict(list)
    indeg = np.zeros(P, int)
    for (u, v, kind, sense, tab) in arcs:
        if kind == "net":
            dl = {(0, 0): elm_of_pin[v], (1, 1): elm_of_pin[v]}
        else:
            dl = {(i, o): max(0.0, const_value(lib, tab + o)) for (i, o) in _pairs(sense)}
        succ[u].append((v, dl))
        indeg[v] += 1
    seed_at = {}
    for k in range(cons.pi_pin.size):
        p = int(cons.pi_pin[k])
        if indeg[p] == 0:
            seed_at[p] = [float(x) for x in cons.pi_at[k]]
    for p in range(P):
        if int(d.pin_role[p]) == ROLE_FF_CK and indeg[p] == 0:
            seed_at[p] = [0.0, T / 2, 0.0, T / 2]
    # arrivals (for the data-arrival condition of the check seeds)
    reach = defaultdict(bool)

    def mark(v, rf):
        if reach[(v, rf)]:
            return
        reach[(v, rf)] = True
        for (w, dl) in succ[v]:
            for (i, o) in dl:
                if i == rf:
                    mark(w, o)
    for s in seed_at:
        for rf in (0, 1):
            mark(s, rf)
    seed = {}
    for k in range(cons.po_pin.size):
        p = int(cons.po_pin[k])
        for rf in (0, 1):
            x = T - float(cons.po_out_max[k, rf]) if late else -float(cons.po_out_min[k, rf])
            old = seed.get((p, rf))
            seed[(p, rf)] = x if old is None else (min(old, x) if late else max(old, x))
    for c in range(d.num_checks):
        p, tb = int(d.chk_d[c]), int(d.chk_tab[c])
        for rf in (0, 1):
            if reach[(p, rf)]:
                x = T - const_value(lib, tb + rf) if late else const_value(lib, tb + 2 + rf)
                old = seed.get((p, rf))
                seed[(p, rf)] = x if old is None else (min(old, x) if late else max(old, x))
    out = []

    def walk(v, rf, acc, nodes, ats):
        nodes.append((v, rf))
        ats.append(acc)
        if (v, rf) in seed:
            sl = seed[(v, rf)] - acc if late else acc - seed[(v, rf)]
            out.append((sl, v, tuple(nodes), tuple(ats)))
        for (w, dl) in succ[v]:
            for (i, o), x in dl.items():
                if i == rf:
                    walk(w, o, acc + x, nodes, ats)
        nodes.pop()
        ats.pop()

    for s, a in seed_at.items():
        for rf in (0, 1):
            walk(s, rf, a[2 + rf] if late else a[rf], [], [])
    out.sort(key=lambda t: (t[0], t[1], tuple(reversed(t[2]))))
    return out


def select_paths(paths, k, nworst, slack_lt=INF):
    """Report selection over a sorted path list: slack < slack_lt, at most
    nworst per endpoint, k in all."""
    kept, cnt = [], defaultdict(int)
    for p in paths:
        if len(kept) >= k or not p[0] < slack_lt:
            break
        if cnt[p[1]] >= nworst:
            continue
        cnt[p[1]] += 1
        kept.append(p)
    return kept


def path_matches(ex, k, pins):
    """a path (pin sequence, startpoint first) matches
    exception k iff its startpoint is in the -from list (if any) and it
    touches one pin of every -through segment in order -- positions
    i_1 <= i_2 <= ... (one pin may serve consecutive segments, X8),
    searched exhaustively."""
    f0, f1 = int(ex.from_ptr[k]), int(ex.from_ptr[k + 1])
    if f1 > f0 and pins[0] not in set(int(x) for x in ex.from_pins[f0:f1]):
        return False
    segs = []
    if ex.thr_ptr is not None:
        for sg in range(int(ex.thr_ptr[k]), int(ex.thr_ptr[k + 1])):
            segs.append(set(int(x) for x in ex.seg_pins[int(ex.seg_ptr[sg]):int(ex.seg_ptr[sg + 1])]))

    def rec(j, lo):
        if j == len(segs):
            return True
        return any(pins[i] in segs[j] and rec(j + 1, i) for i in range(lo, len(pins)))
    return rec(0, 0)


def path_tag(ex, pins):
    """bit k: the path matches exception k's -from / -through requirements"""
    return sum(1 << k for k in range(ex.num) if path_matches(ex, k, pins))


def exception_of(ex, tag, e, late):
    """The exception a path of startpoint tag `tag` (bitset over ex) meets at
    endpoint e, for the late (setup) or early (hold) check: DESIGN.md X2-X3
    precedence -- false path, then max (late) / min (early) delay, then
    multicycle; the first listed of a kind.  -> (mode, value): mode 0 shift,
    1 replace, 2 no check; None without exception."""
    cand = {0: None, 2 if late else 3: None, 1: None}
    for k in range(ex.num):
        f0, f1 = int(ex.from_ptr[k]), int(ex.from_ptr[k + 1])
        t0, t1 = int(ex.to_ptr[k]), int(ex.to_ptr[k + 1])
        has_thr = ex.thr_ptr is not None and int(ex.thr_ptr[k + 1]) > int(ex.thr_ptr[k])
        if (f1 > f0 or has_thr) and not (tag >> k) & 1:
            continue
        if t1 > t0 and e not in set(int(x) for x in ex.to_pins[t0:t1]):
            continue
        kk = int(ex.kind[k])
        if kk in cand and cand[kk] is None:
            cand[kk] = k
    return cand


def path_slacks_with_exceptions(d, elm_of_pin):
    """Frozen-delay brute force of the timing exceptions (d.exceptions):
    every startpoint -> endpoint path is enumerated; a path's required time
    is its endpoint's seed modified by the exception of (the exceptions its
    pin sequence matches, path_tag; its endpoint); the setup / hold slack of a (pin, rf) is the minimum over
    the complete paths through it, an endpoint's worst slack the minimum over
    the paths ending there (false paths excluded).  Returns slack [P][4] and
    res (WNS_s, TNS_s, WNS_h, TNS_h)."""
    lib = d.libs[0]
    cons = d.cons
    ex = d.exceptions
    T = float(cons.period)
    ck = getattr(d, "clocks", None)

    def clk_of(p):
        return int(ck.pin_clk[p]) if ck is not None else 0

    def per(c):
        return float(ck.period[c]) if ck is not None else T

    def rel(tl, tc):
        """(setup, hold) relationship: first 1000 launch edges, next capture edge."""
        s, h = INF, -INF
        for i in range(1000):
            a = i * tl
            nxt = (math.floor(a / tc) + 1.0) * tc
            s, h = min(s, nxt - a), max(h, nxt - tc - a)
        return s, h
    arcs = _fanin_lists(d)
    P = d.num_pins
    succ = defaultdict(list)
    indeg = np.zeros(P, int)
    for (u, v, kind, sense, tab) in arcs:
        if kind == "net":
            dl = {(0, 0): elm_of_pin[v], (1, 1): elm_of_pin[v]}
        else:
            dl = {(i, o): max(0.0, const_value(lib, tab + o)) for (i, o) in _pairs(sense)}
        succ[u].append((v, dl))
        indeg[v] += 1
    seed_at = {}
    for k in range(cons.pi_pin.size):
        p = int(cons.pi_pin[k])
        if indeg[p] == 0:
            seed_at[p] = [float(x) for x in cons.pi_at[k]]
    for p in range(P):
        if int(d.pin_role[p]) == ROLE_FF_CK and indeg[p] == 0:
            tc = per(clk_of(p))
            seed_at[p] = [0.0, tc / 2, 0.0, tc / 2]
    cap_clk = {}
    for k in range(cons.po_pin.size):
        cap_clk[int(cons.po_pin[k])] = clk_of(int(cons.po_pin[k]))
    for c in range(d.num_checks):
        cap_clk[int(d.chk_d[c])] = clk_of(int(d.chk_ck[c]))
    base_l = defaultdict(lambda: [INF, INF])
    base_e = defaultdict(lambda: [-INF, -INF])
    po_l, po_e, ck_l, ck_e = {}, {}, {}, {}
    for k in range(cons.po_pin.size):
        p = int(cons.po_pin[k])
        po_l.setdefault(p, []).append([T - float(cons.po_out_max[k, rf]) for rf in (0, 1)])
        po_e.setdefault(p, []).append([-float(cons.po_out_min[k, rf]) for rf in (0, 1)])
    for c in range(d.num_checks):
        p, tb = int(d.chk_d[c]), int(d.chk_tab[c])
        ck_l.setdefault(p, []).append([T - const_value(lib, tb + rf) for rf in (0, 1)])
        ck_e.setdefault(p, []).append([const_value(lib, tb + 2 + rf) for rf in (0, 1)])
    endpoints = sorted(set(po_l) | set(ck_l))

    def mod(v, ov):
        if ov is None:
            return v
        mode, val = ov
        return INF if mode == 2 else (val if mode == 1 else v + val)

    def req(e, rf, tg, late, s_clk=0):
        # the clock relationship of (launch, capture) replaces the single-clock
        # setup edge T / hold edge 0 of the base seeds
        tcap = per(cap_clk.get(e, 0))
        rs, rh = rel(per(s_clk), tcap)
        shift = (rs - T) if late else rh
        c = exception_of(ex, tg, e, late) if ex is not None else {0: None, 1: None, 2: None, 3: None}
        ov = (0, shift)
        if c[0] is not None:
            ov = (2, 0.0)
        elif c[2 if late else 3] is not None:
            ov = (1, float(ex.value[c[2 if late else 3]]))
        elif c[1] is not None:
            ov = (0, shift + (float(ex.value[c[1]]) - 1.0) * tcap)
        vals = [x[rf] for x in (po_l if late else po_e).get(e, [])] + [x[rf] for x in (ck_l if late else ck_e).get(e, [])]
        if not vals:
            return None
        if late:
            return min(mod(x, ov) for x in vals)
        r = [mod(x, ov) for x in vals]
        r = [(-INF if ov is not None and ov[0] == 2 else x) for x in r]
        return max(r)

    slack = np.full((P, 4), INF)
    ws = {e: INF for e in endpoints}
    wh = {e: INF for e in endpoints}

    def walk(stack, v, rf, acc, s, s_rf):
        stack.append((v, rf))
        if v in po_l or v in ck_l:
            tg = path_tag(ex, [x for (x, _) in stack]) if ex is not None else 0
            rl = req(v, rf, tg, True, clk_of(s))
            if rl is not None and rl < INF:
                sl = rl - (seed_at[s][2 + s_rf] + acc)
                ws[v] = min(ws[v], sl)
                for (x, r) in stack:
                    slack[x, 2 + r] = min(slack[x, 2 + r], sl)
            re = req(v, rf, tg, False, clk_of(s))
            if re is not None and re > -INF:
                sh = (seed_at[s][s_rf] + acc) - re
                wh[v] = min(wh[v], sh)
                for (x, r) in stack:
                    slack[x, r] = min(slack[x, r], sh)
        for (w, dl) in succ[v]:
            for (i, o), x in dl.items():
                if i == rf:
                    walk(stack, w, o, acc + x, s, s_rf)
        stack.pop()

    for s in seed_at:
        for rf in (0, 1):
            walk([], s, rf, 0.0, s, rf)
    wsv = [ws[e] for e in endpoints]
    whv = [wh[e] for e in endpoints]
    res = (min(wsv, default=INF), sum(min(0.0, x) for x in wsv if x < INF),
           min(whv, default=INF), sum(min(0.0, x) for x in whv if x < INF))
    return slack, res
