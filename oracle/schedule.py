"""Pure-Python restatement of the reference schedule path -- TEST ORACLE ONLY.

Nothing in the product imports this module; tests/ and bench.py's CPU
baseline use it as a checker.  It follows the reference algorithm statement
by statement (file:line under /root/reference/proj) and is pinned in
tests/test_oracle.py against the reference's 5 byte-frozen goldens and the
oracle/_ref grid fixtures (tests/golden/).  Pure-Python loops: small cases only.
"""
from fractions import Fraction

GPIPE, DAPPLE, CHIMERA, CHIMERA_WAVE, HANAYO = range(5)
FORWARD, BACKWARD, SEND, RECEIVE, BATCHED_EXCHANGE, OPTIMIZER_STEP = range(6)
ACTIVATION, GRADIENT = 0, 1
DOWN, UP = 0, 1
SCHEME_NAMES = ["gpipe", "dapple", "chimera", "chimera-wave", "hanayo"]


def is_wave(scheme):
    return scheme in (HANAYO, CHIMERA_WAVE)


def make_config(scheme, P, B, W=1, D=1):
    """src/config.cpp:47-81."""
    if P < 1 or B < 1 or W < 1 or D < 1:
        raise ValueError("sizes must be positive")
    if B < P:
        raise ValueError("B must be >= P")
    if scheme in (CHIMERA, CHIMERA_WAVE) and (P % 2 or B % 2):
        raise ValueError("P and B must be even")
    if not is_wave(scheme) and W > 1:
        raise ValueError("W must be 1")
    return dict(scheme=scheme, P=P, B=B, W=W, D=D, S=2 * W * P if is_wave(scheme) else P)


def make_placement(cfg):
    """src/placement.cpp:22-83: per device, list of (index, fraction, direction)."""
    P, W, sch = cfg["P"], cfg["W"], cfg["scheme"]
    if sch in (GPIPE, DAPPLE):
        return [[(p, Fraction(1), DOWN)] for p in range(P)]
    if sch == CHIMERA:
        return [[(p, Fraction(1), DOWN), (P - 1 - p, Fraction(1), UP)] for p in range(P)]
    out = []
    for p in range(P):
        row = []
        for w in range(W):
            base = 2 * w * P
            row.append((base + p, Fraction(1, 2 * W), DOWN))
            row.append((base + 2 * P - 1 - p, Fraction(1, 2 * W), UP))
        out.append(row)
    return out


def microbatch_direction(cfg, b):
    """src/action.cpp:85-89."""
    if cfg["scheme"] != CHIMERA:
        return DOWN
    return DOWN if b < (cfg["B"] + 1) // 2 else UP


def slice_owner(cfg, placement, s, direction):
    """src/action.cpp:91-102."""
    for d, row in enumerate(placement):
        for r, (idx, _, dr) in enumerate(row):
            if idx != s:
                continue
            if cfg["scheme"] == CHIMERA and dr != direction:
                continue
            return d, r
    return -1, -1


def _chains(cfg, placement):
    """src/schedule.cpp:42-57."""
    return [[slice_owner(cfg, placement, s, microbatch_direction(cfg, b)) for s in range(cfg["S"])]
            for b in range(cfg["B"])]


def generate_compute_order(cfg, placement, cost):
    """GreedyScheduler::run, src/schedule.cpp:60-312 (full rescan, as the reference)."""
    P, B, S, sch = cfg["P"], cfg["B"], cfg["S"], cfg["scheme"]
    tf, tb, tc = cost
    wave = is_wave(sch)
    fdur = tf / (2.0 * cfg["W"]) if wave else tf
    bdur = tb / (2.0 * cfg["W"]) if wave else tb
    ch = _chains(cfg, placement)
    NONE = -1.0
    fwd_end = [[NONE] * S for _ in range(B)]
    bwd_end = [[NONE] * S for _ in range(B)]
    engine = [0.0] * P
    streams = [[] for _ in range(P)]
    fwd_started = [[0, 0] for _ in range(P)]
    bwd_done = [[0, 0] for _ in range(P)]
    fwd_done_count = [0] * P
    fwd_total = [0] * P
    for b in range(B):
        for s in range(S):
            fwd_total[ch[b][s][0]] += 1
    entered, exited = [0, 0], [0, 0]
    dir_id = [0 if microbatch_direction(cfg, b) == DOWN else 1 for b in range(B)]

    def started_here(b, s):  # :144-154
        return any(ch[b][q][0] == ch[b][s][0] and fwd_end[b][q] != NONE for q in range(s))

    def admissible_fwd(dev, b, s):  # :118-140
        dr = dir_id[b]
        if sch == GPIPE:
            return True
        if sch in (DAPPLE, CHIMERA):
            pos = P - 1 - dev if (sch == CHIMERA and dr == 1) else dev
            if sch == CHIMERA:
                down = (B + 1) // 2
                cnt = down if dr == 0 else B - down
            else:
                cnt = B
            cap = min(P - pos, cnt)
            return fwd_started[dev][dr] - bwd_done[dev][dr] < cap or started_here(b, s)
        if s != 0:
            return True
        return entered[dr] - exited[dr] < P

    def arrival(bw, b, s):  # :167-184
        if not bw:
            if s == 0:
                return 0.0
            prod = fwd_end[b][s - 1]
            if prod == NONE:
                return NONE
            return prod + (tc if ch[b][s - 1][0] != ch[b][s][0] else 0.0)
        if s == S - 1:
            return fwd_end[b][s]
        prod = bwd_end[b][s + 1]
        if prod == NONE:
            return NONE
        return prod + (tc if ch[b][s + 1][0] != ch[b][s][0] else 0.0)

    def policy_less(x, y):  # :190-198
        if x[0] != y[0]:
            return x[0]
        rx = x[2] if x[0] else S - 1 - x[2]
        ry = y[2] if y[0] else S - 1 - y[2]
        if rx != ry:
            return rx < ry
        if x[1] != y[1]:
            return x[1] < y[1]
        if x[2] != y[2]:
            return x[2] > y[2] if x[0] else x[2] < y[2]
        return False

    for _ in range(2 * B * S):  # :85-93, schedule_one :200-278
        found, best_start, best_dev, best = False, 0.0, -1, None
        for dev in range(P):
            ready = []
            for b in range(B):
                for s in range(S):
                    if ch[b][s][0] != dev:
                        continue
                    if fwd_end[b][s] == NONE:
                        a = arrival(False, b, s)
                        if a != NONE and admissible_fwd(dev, b, s):
                            ready.append((a, (False, b, s)))
                    elif bwd_end[b][s] == NONE:
                        if s + 1 < S and bwd_end[b][s + 1] == NONE:
                            continue
                        a = arrival(True, b, s)
                        ok = fwd_done_count[dev] == fwd_total[dev] if sch == GPIPE else True
                        if a != NONE and ok:
                            ready.append((a, (True, b, s)))
            if not ready:
                continue
            start = min(max(engine[dev], a) for a, _ in ready)
            pick = None
            for a, n in ready:
                if a > start:
                    continue
                if pick is None or policy_less(n, pick):
                    pick = n
            if not found or start < best_start or (start == best_start and dev < best_dev):
                found, best_start, best_dev, best = True, start, dev, pick
        if not found:
            raise RuntimeError("schedule generation stalled with work remaining")
        bw, b, s = best
        end = best_start + (bdur if bw else fdur)
        engine[best_dev] = end
        streams[best_dev].append(best)
        dr = dir_id[b]
        first_visit = not any(ch[b][q][0] == best_dev for q in range(s))
        if not bw:
            fwd_end[b][s] = end
            fwd_done_count[best_dev] += 1
            if first_visit:
                fwd_started[best_dev][dr] += 1
            if s == 0:
                entered[dr] += 1
        else:
            bwd_end[b][s] = end
            if first_visit:
                bwd_done[best_dev][dr] += 1
            if s == 0:
                exited[dr] += 1
    return streams


def _key(a):
    """Message key (payload, microbatch, low slice): src/schedule.cpp:384-418."""
    kind, mb, _, s, _, payload, _ = a
    sending = kind in (SEND, BATCHED_EXCHANGE)
    if payload == ACTIVATION:
        low = s if sending else s - 1
    else:
        low = s - 1 if sending else s
    return (payload, mb, low)


def insert_comm(cfg, placement, streams):
    """src/schedule.cpp:333-473.  Actions are 7-tuples
    (kind, microbatch, local_module_rank, slice_index, peer, payload, batch_group)."""
    ch = _chains(cfg, placement)
    P, S = cfg["P"], cfg["S"]
    full = [[] for _ in range(P)]
    for dev in range(P):
        for bw, b, s in streams[dev]:
            src = s + 1 if bw else s - 1
            dst = s - 1 if bw else s + 1
            pay = GRADIENT if bw else ACTIVATION
            lr = ch[b][s][1]
            if 0 <= src < S and ch[b][src][0] != dev:
                full[dev].append((RECEIVE, b, lr, s, ch[b][src][0], pay, -1))
            full[dev].append((BACKWARD if bw else FORWARD, b, lr, s, -1, -1, -1))
            if 0 <= dst < S and ch[b][dst][0] != dev:
                full[dev].append((SEND, b, lr, s, ch[b][dst][0], pay, -1))
    send_at, recv_at = {}, {}
    for dev in range(P):
        for i, a in enumerate(full[dev]):
            if a[0] == SEND:
                send_at[_key(a)] = (dev, i)
            elif a[0] == RECEIVE:
                recv_at[_key(a)] = (dev, i)
    group = [[-1] * len(full[d]) for d in range(P)]
    nxt = 0
    for dev in range(P):
        st = full[dev]
        for i in range(len(st) - 1):
            a, b = st[i], st[i + 1]
            if group[dev][i] >= 0 or group[dev][i + 1] >= 0:
                continue
            opposing = (a[0] == SEND and b[0] == RECEIVE) or (a[0] == RECEIVE and b[0] == SEND)
            if not opposing or a[4] != b[4] or a[4] < 0:
                continue
            snd, rcv = (a, b) if a[0] == SEND else (b, a)
            pr = recv_at[_key(snd)]
            # the peer's send of the message this device receives
            ps = send_at[_key(rcv)]
            q = a[4]
            if pr[0] != q or ps[0] != q or abs(pr[1] - ps[1]) != 1:
                continue
            if group[q][pr[1]] >= 0 or group[q][ps[1]] >= 0:
                continue
            group[dev][i] = group[dev][i + 1] = nxt
            group[q][pr[1]] = group[q][ps[1]] = nxt
            nxt += 1
    out = []
    for dev in range(P):
        st, row, i = full[dev], [], 0
        while i < len(st):
            g = group[dev][i]
            if g < 0:
                row.append(st[i])
                i += 1
                continue
            snd = st[i] if st[i][0] == SEND else st[i + 1]
            row.append((BATCHED_EXCHANGE,) + snd[1:6] + (g,))
            i += 2
        row.append((OPTIMIZER_STEP, -1, -1, -1, -1, -1, -1))
        out.append(row)
    return out


def generate_schedule(cfg, cost=(1.0, 2.0, 0.0)):
    """src/schedule.cpp:475-499 (with make_placement)."""
    pl = make_placement(cfg)
    return insert_comm(cfg, pl, generate_compute_order(cfg, pl, cost)), pl


def simulate(cfg, actions, cost=(1.0, 2.0, 0.0)):
    """src/simulate.cpp:57-178 -> (makespan, intervals, comm_events)."""
    tf, tb, tc = cost
    wave = is_wave(cfg["scheme"])
    fdur = tf / (2.0 * cfg["W"]) if wave else tf
    bdur = tb / (2.0 * cfg["W"]) if wave else tb
    P = len(actions)
    groups = {}
    for d in range(P):
        for i, a in enumerate(actions[d]):
            if a[0] == BATCHED_EXCHANGE:
                groups.setdefault(a[6], []).append((d, i))
    fire, reached = {}, {}
    pc = [0] * P
    clock = [0.0] * P
    last_start = [0.0] * P
    pending = [0.0] * P
    intervals = [[] for _ in range(P)]
    events = []
    progressed = True
    while progressed:
        progressed = False
        for d in range(P):
            while pc[d] < len(actions[d]):
                a = actions[d][pc[d]]
                k = a[0]
                if k in (FORWARD, BACKWARD):
                    start = max(clock[d], pending[d])
                    end = start + (fdur if k == FORWARD else bdur)
                    intervals[d].append((pc[d], k, a[1], a[3], start, end))
                    clock[d], last_start[d], pending[d] = end, start, 0.0
                elif k == OPTIMIZER_STEP:
                    pass
                elif k == SEND:
                    fire[_key(a)] = clock[d]
                elif k == RECEIVE:
                    f = fire.get(_key(a))
                    if f is None:
                        break
                    arr = max(last_start[d], f) + tc
                    pending[d] = max(pending[d], arr)
                    events.append((a[4], d, last_start[d], arr))
                else:
                    reached[(d, pc[d])] = clock[d]
                    m = groups[a[6]]
                    other = m[1] if m[0] == (d, pc[d]) else m[0]
                    if other not in reached:
                        break
                    start = max(clock[d], reached[other])
                    end = start + tc
                    intervals[d].append((pc[d], k, a[1], a[3], start, end))
                    events.append((d, a[4], start, end))
                    clock[d] = end
                pc[d] += 1
                progressed = True
    for d in range(P):
        if pc[d] < len(actions[d]):
            raise RuntimeError(f"simulation stalled: device {d}")
    events.sort(key=lambda e: (e[3], e[2], e[0], e[1]))
    return max(clock), intervals, events


def bubble_ratio(makespan, intervals):
    """src/analytics.cpp:32-46."""
    busy = 0.0
    for dev in intervals:
        for iv in dev:
            if iv[1] in (FORWARD, BACKWARD):
                busy += iv[5] - iv[4]
    return 1.0 - busy / (len(intervals) * makespan)


def memory_profile(placement, intervals):
    """src/analytics.cpp:48-91 -> (weights, peaks) as Fractions."""
    weights, peaks = [], []
    for d, row in enumerate(placement):
        frac = {idx: f for idx, f, _ in row}
        weights.append(sum((f for _, f, _ in row), Fraction(0)))
        ev = []
        for iv in intervals[d]:
            if iv[1] == BATCHED_EXCHANGE:
                continue
            f = frac[iv[3]]
            ev.append((iv[4], f) if iv[1] == FORWARD else (iv[5], -f))
        ev.sort()
        live = peak = Fraction(0)
        for _, delta in ev:
            live += delta
            peak = max(peak, live)
        peaks.append(peak)
    return weights, peaks


def analytic_bubble_hanayo(P, W, tf, tb, tc):
    """Eq. 1, src/analytics.cpp:124-141 (exact)."""
    tf, tb, tc = Fraction(tf), Fraction(tb), Fraction(tc)
    num = tb / W + (1 + 2 * W + Fraction(2, P) + Fraction(P - 2, 3)) * tc
    den = Fraction(P, P - 1) * tf + (Fraction(1, 2 * W) + Fraction(P, P - 1)) * tb + \
        (Fraction(P - 2, 2) + 4 * W) * tc
    return num / den


def analytic_bubble_simplified(P, W):
    """src/analytics.cpp:159-164."""
    return Fraction(2 * P - 2, 3 * P * W + P - 1)
