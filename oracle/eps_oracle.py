"""CPU restatement of the reference's decision path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import it.  The
product computes the same decisions in C++ (libeps_b200.so).

Every function restates the algorithm of the reference artifact
(/root/reference/proj, arXiv 2102.03161's control plane) and cites the file
and lines it follows.  Pinned against (a) the reference's own known-answer
tests (tests/test_oracle_golden.py: test_freeze.cpp, test_autopipe.cpp,
test_autodp.cpp, test_autocache.cpp, test_engine.cpp, test_model.cpp) and
(b) outputs of the reference itself compiled from its sources
(oracle/_ref/libeps_ref.so, fixtures in tests/golden/).

Floating-point expressions keep the reference's operand order: Python floats
are IEEE binary64 like C++ doubles, so the same order gives the same bits.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


# ---- rng.hpp:11-43 ----------------------------------------------------------
class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:  # rng.hpp:15-20
        self.state = (self.state + GOLDEN) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def next_below(self, bound: int) -> int:  # rng.hpp:24
        return self.next() % bound

    def next_unit(self) -> float:  # rng.hpp:27
        return float(self.next() >> 11) * 2.0 ** -53


def hash_combine(a: int, b: int) -> int:  # rng.hpp:33-36
    a &= MASK64
    b &= MASK64
    return a ^ ((b + GOLDEN + ((a << 6) & MASK64) + (a >> 2)) & MASK64)


def deterministic_shuffle(v: list, rng: SplitMix64) -> None:  # rng.hpp:38-43
    for i in range(len(v), 1, -1):
        j = rng.next_below(i)
        v[i - 1], v[j] = v[j], v[i - 1]


# ---- model.cpp ---------------------------------------------------------------
@dataclass
class Model:
    attention: List[int]
    mlp: List[int]
    act: List[int]
    bytes_per_param: int = 4

    @property
    def L(self) -> int:
        return len(self.attention)

    def prefix(self, layer: int) -> int:  # model.cpp:17-22
        if layer < 0 or layer > self.L:
            raise ValueError("prefix_params: layer out of range")
        return sum(self.attention[i] + self.mlp[i] for i in range(layer))

    def total(self) -> int:
        return self.prefix(self.L)


def att_block(d: int) -> int:  # model.cpp:109-114
    return 3 * (d * d + d) + (d * d + d) + 2 * d


def mlp_block(d: int, f: int) -> int:  # model.cpp:116-121
    return (d * f + f) + (f * d + d) + 2 * d


def vit_model(layers=12, d=768, f=3072, image=224, patch=16, channels=3, classes=1000) -> Model:
    """model.cpp:125-150 generalised to any ViT geometry."""
    tokens = (image // patch) ** 2 + 1
    att = [att_block(d)] * layers
    mlp = [mlp_block(d, f)] * layers
    att[0] += d * (patch * patch * channels) + d + d + tokens * d
    mlp[-1] += d * classes + classes
    act = [tokens * d * 4] * (2 * layers + 1)
    act[0] = image * image * channels * 4
    return Model(att, mlp, act)


def bert_model(layers=24, d=1024, f=4096, seq=512, positions=512, vocab=30522,
               head=None) -> Model:
    """model.cpp:152-179 generalised (head defaults to pooler + QA span head)."""
    if head is None:
        head = (d * d + d) + (d * 2 + 2)
    att = [att_block(d)] * layers
    mlp = [mlp_block(d, f)] * layers
    att[0] += vocab * d + positions * d + 2 * d + 2 * d
    mlp[-1] += head
    act = [seq * d * 4] * (2 * layers + 1)
    act[0] = seq * 8
    return Model(att, mlp, act)


@dataclass
class Seq:  # SublayerSeq, model.hpp:66-74
    params: List[int]
    gidx: List[int]
    frozen_params: int = 0
    frozen_layers: int = 0

    def active(self) -> int:
        return sum(self.params)


def m_partition(m: Model, l_frozen: int) -> Seq:  # model.cpp:79-92
    if l_frozen < 0 or l_frozen > m.L:
        raise ValueError("m_partition: frozen layer count out of [0, L]")
    p, g = [], []
    for i in range(l_frozen, m.L):
        p += [m.attention[i], m.mlp[i]]
        g += [2 * i, 2 * i + 1]
    return Seq(p, g, m.prefix(l_frozen), l_frozen)


# ---- freeze.cpp --------------------------------------------------------------
class FreezeState:
    def __init__(self, alpha: float):
        if not (0.0 < alpha < 1.0):
            raise ValueError("freeze: alpha must be in (0,1)")
        self.alpha = alpha
        self.history: List[Tuple[int, int, float]] = []

    def frozen_count(self) -> int:
        return self.history[-1][1] if self.history else 0


def next_frozen_count(st: FreezeState, norms: Sequence[float], L: int) -> int:
    """freeze.cpp:22-50 (Eq. 1)."""
    if len(norms) != L:
        raise ValueError("freeze: gradient norm vector length mismatch")
    for g in norms:
        if g < 0.0 or not math.isfinite(g):
            raise ValueError("freeze: gradient norms must be finite and >= 0")
    prev = st.frozen_count()
    bound = prev + st.alpha * (L - prev)
    argmin = prev
    for l in range(prev, L):
        if norms[l] < norms[argmin]:
            argmin = l
    result = prev
    if prev < L:
        result = int(math.floor(min(bound, float(argmin))))
        result = max(prev, min(result, L))
    t = 1 if not st.history else st.history[-1][0] + 1
    st.history.append((t, result, bound))
    return result


def frozen_bound_closed_form(T: int, L: int, alpha: float) -> float:  # freeze.cpp:52-60
    if not (0.0 < alpha < 1.0):
        raise ValueError("frozen_bound_closed_form: alpha must be in (0,1)")
    al = alpha * L
    s = al / (1.0 - alpha)
    for t in range(2, T + 1):
        s += al / math.pow(1.0 - alpha, t)
    return math.pow(1.0 - alpha, T) * s


def synthetic_norms(profile: int, seed: int, L: int, switchover: int, epoch: int) -> List[float]:
    """SyntheticNormSource::at_epoch, freeze.cpp:121-152 (profile 1 = early-random)."""
    decay = math.pow(0.9, epoch)
    random_phase = profile == 1 and epoch < switchover
    out = []
    for l in range(L):
        rng = SplitMix64(hash_combine(hash_combine(seed, epoch), l))
        jitter = rng.next_unit()
        if random_phase:
            out.append(decay * (0.8 + 0.4 * jitter))
        else:
            shape = 1.0 + float(L - 1 - l) / L
            out.append(decay * shape * (1.0 + 0.02 * jitter))
    if random_phase:
        rng = SplitMix64(hash_combine(seed, (0x5EED + epoch) & MASK64))
        quarter = max(1, L // 4)
        j = L - 1 - rng.next_below(quarter)
        out[j] *= 0.05
    return out


# ---- autopipe.cpp ------------------------------------------------------------
@dataclass
class Plan:
    K: int
    spans: List[Tuple[int, int]]
    param_sums: List[int]
    eff: List[float]
    frozen_params: int
    frozen_layers: int

    def max_eff(self) -> float:
        m = 0.0
        for e in self.eff:
            m = max(m, e)
        return m


def _popvar(params: List[int], begin: int) -> float:  # autopipe.cpp:37-51
    n = len(params) - begin
    if n <= 0:
        return 0.0
    mean = 0.0
    for i in range(begin, len(params)):
        mean += float(params[i])
    mean /= n
    var = 0.0
    for i in range(begin, len(params)):
        d = float(params[i]) - mean
        var += d * d
    return var / n


def load_balance(seq: Seq, K: int, lam: float, criterion: int = 0) -> Plan:
    """autopipe.cpp:55-122 -- greedy fill, accept on <= (autopipe.cpp:100)."""
    n = len(seq.params)
    if K < 1 or (n == 0 and K != 1) or (n > 0 and K > n):
        raise ValueError("load_balance: infeasible K")
    frozen_share = lam * float(seq.frozen_params)
    remaining = float(seq.active())
    assigned = 0
    spans, sums, effs = [], [], []
    for k in range(K):
        begin = assigned
        left = K - k
        mean = remaining / left
        pv = _popvar(seq.params, assigned)
        slack = pv / left if criterion == 1 else math.sqrt(pv) / left
        target = mean + slack
        start_eff = frozen_share if k == 0 else 0.0
        eff, raw, count = start_eff, 0, 0
        while assigned < n:
            if k < K - 1:
                if n - assigned <= left - 1:
                    break
                fits = eff + float(seq.params[assigned]) <= target
                if not fits:
                    if count > 0:
                        break
                    if start_eff > target:
                        break
            cand = float(seq.params[assigned])
            eff += cand
            raw += seq.params[assigned]
            remaining -= cand
            assigned += 1
            count += 1
        spans.append((begin, assigned))
        sums.append(raw)
        effs.append((frozen_share if k == 0 else 0.0) + float(raw))
    return Plan(K, spans, sums, effs, seq.frozen_params, seq.frozen_layers)


def try_compress(seq: Seq, k: int, lam: float, m_gpu0: float, criterion: int = 0):
    """autopipe.cpp:124-158 -- halve while max_eff(K/2) <= M_GPU^(0)."""
    if k < 1 or (k & (k - 1)) != 0:
        raise ValueError("try_compress: K must be a power of two")
    if not seq.params:
        return 1, load_balance(seq, 1, lam, criterion), []
    plan = load_balance(seq, k, lam, criterion)
    attempts = []
    while k >= 2:
        half = k // 2
        if half > len(seq.params):
            break
        cand = load_balance(seq, half, lam, criterion)
        me = cand.max_eff()
        attempts.append((k, me))
        if me <= m_gpu0:
            k, plan = half, cand
        else:
            break
    return k, plan, attempts


# ---- cost_model.cpp / schedule.cpp / chunks.cpp ------------------------------
@dataclass
class Cost:
    c_fwd: float = 0.035 / (12.0e6 * 300.0)
    backward_ratio: float = 2.0
    c_update: float = 1.0e-11
    per_microbatch_overhead: float = 2.0e-4
    allreduce_bucket_bytes: float = 25.0e6
    comm_latency: float = 0.0
    transition_overheads: Dict[str, float] = field(default_factory=dict)


def ring_allreduce_time(nbytes, width, bw, lat):  # cost_model.cpp:42-47
    if width < 2:
        return 0.0
    factor = 2.0 * (width - 1) / float(width)
    return factor * nbytes / bw + lat


def build_schedule(stages, M, batch, R, spans_nodes, intra, inter, bpp, cm: Cost,
                   integer_mb=False) -> dict:
    """schedule.cpp:19-199; stages = [(fwd, bwd, prefix_s, in_bytes)]."""
    K = len(stages)
    sizes = [batch / M] * M
    if integer_mb:
        b = int(round(batch))
        sizes = [float(b // M + (1 if i < b % M else 0)) for i in range(M)]
    f_end = [[0.0] * M for _ in range(K)]
    b_end = [[0.0] * M for _ in range(K)]
    busy = [0.0] * K
    free = [0.0] * K
    xfer_total = 0.0

    def fwd(d, b):
        f, _, pre, _ = stages[d]
        work = (cm.c_fwd * f + pre) * sizes[b]
        return work + (cm.per_microbatch_overhead if (f > 0 or pre > 0) else 0.0)

    def bwd(d, b):
        bw = stages[d][1]
        if bw <= 0:
            return 0.0
        return cm.backward_ratio * cm.c_fwd * bw * sizes[b] + cm.per_microbatch_overhead

    for b in range(M):
        for d in range(K):
            ready = 0.0
            if d > 0:
                x = stages[d][3] * sizes[b] / intra + cm.comm_latency
                ready = f_end[d - 1][b] + x
                if x > 0:
                    xfer_total += x
            start = max(ready, free[d])
            dur = fwd(d, b)
            f_end[d][b] = start + dur
            free[d] = f_end[d][b]
            if dur > 0:
                busy[d] += dur
    first = K
    for d in range(K):
        if stages[d][1] > 0:
            first = d
            break
    has_bwd = first < K
    if has_bwd:
        for d in range(first, K):
            free[d] = f_end[d][M - 1]
        for b in range(M - 1, -1, -1):
            for d in range(K - 1, first - 1, -1):
                ready = 0.0
                if d < K - 1:
                    x = stages[d + 1][3] * sizes[b] / intra + cm.comm_latency
                    ready = b_end[d + 1][b] + x
                    if x > 0:
                        xfer_total += x
                start = max(ready, free[d])
                dur = bwd(d, b)
                b_end[d][b] = start + dur
                free[d] = b_end[d][b]
                if dur > 0:
                    busy[d] += dur
    cms = 0.0
    for d in range(K):
        cms = max(cms, f_end[d][M - 1])
        if has_bwd and d >= first:
            cms = max(cms, b_end[d][0])
    bubbles = [cms - busy[d] for d in range(K)]
    buckets = []
    if R >= 2 and has_bwd:
        cap = cm.allreduce_bucket_bytes
        cur = None
        for d in range(K - 1, first - 1, -1):
            rem = stages[d][1] * bpp
            while rem > 0:
                if cur is None:
                    cur = [0.0, d, b_end[d][0]]
                cur[1] = d
                cur[2] = max(cur[2], b_end[d][0])
                take = min(cap - cur[0], rem)
                cur[0] += take
                rem -= take
                if cur[0] >= cap:
                    buckets.append(cur)
                    cur = None
        if cur is not None and cur[0] > 0:
            buckets.append(cur)
    link = inter if spans_nodes else intra
    ar_end = [0.0] * K
    track = 0.0
    ar_total = 0.0
    for nbytes, lowest, ready in buckets:
        dur = ring_allreduce_time(nbytes, R, link, cm.comm_latency)
        start = max(ready, track)
        track = start + dur
        ar_total += dur
        for d in range(lowest, K):
            ar_end[d] = max(ar_end[d], track)
    ms, ms_no = cms, cms
    if has_bwd:
        for d in range(first, K):
            u = cm.c_update * stages[d][1]
            if u <= 0:
                continue
            start = max(b_end[d][0], ar_end[d])
            ms = max(ms, start + u)
            ms_no = max(ms_no, b_end[d][0] + u)
    ms = max(ms, track)
    return dict(makespan=ms, compute_makespan=cms, makespan_without_ar=ms_no,
                bubble_per_device=bubbles, total_bubble=sum_in_order(bubbles),
                allreduce_seconds=ar_total, transfer_seconds=xfer_total,
                exposed_comm=ms - ms_no)


def sum_in_order(xs):
    s = 0.0
    for x in xs:
        s += x
    return s


def stage_loads(plan: Plan, m: Model, seq: Seq, cache_enabled: bool, read_ps: float,
                cm: Cost):
    """schedule.cpp:201-231."""
    out = []
    n = len(seq.params)
    for d in range(plan.K):
        f = float(plan.param_sums[d])
        if d == 0:
            pre = read_ps if cache_enabled else cm.c_fwd * float(plan.frozen_params)
            out.append((f, f, pre, 0.0))
        else:
            b = plan.spans[d][0]
            g = seq.gidx[b] if b < n else 2 * m.L
            out.append((f, f, 0.0, float(m.act[g])))
    return out


def schedule_iteration(plan, m, seq, M, batch, R, cluster, cm, cache_enabled, read_ps):
    """schedule.cpp:233-253; cluster = dict(nodes, intra, inter)."""
    st = stage_loads(plan, m, seq, cache_enabled, read_ps, cm)
    return build_schedule(st, M, batch, R, cluster["nodes"] >= 2, cluster["intra"],
                          cluster["inter"], m.bytes_per_param, cm)


def optimal_chunks(plan, m, seq, batch, R, cluster, cm, cache_enabled=False, read_ps=0.0):
    """chunks.cpp:5-24 -- strict argmin, ties to the smallest M."""
    best_m, best_t, times = None, 0.0, []
    for M in range(plan.K, 6 * plan.K + 1):
        t = schedule_iteration(plan, m, seq, M, batch, R, cluster, cm, cache_enabled,
                               read_ps)["makespan"]
        times.append(t)
        if best_m is None or t < best_t:
            best_m, best_t = M, t
    return best_m, times


# ---- autodp.cpp ----------------------------------------------------------------
def active_ranks(nodes: int, gpn: int, K: int) -> List[int]:  # autodp.cpp:23-40
    return [r for r in range(nodes * gpn) if (r % gpn) % K == 0]


def transition(nodes: int, gpn: int, old_k: int, new_k: int) -> List[Tuple[int, int]]:
    """autodp.cpp:81-111 -> (sender, receiver) pairs."""
    if new_k > old_k:
        raise ValueError("transition: shrinking data-parallel width is unsupported")
    if new_k < 1 or gpn % new_k != 0:
        raise ValueError("transition: new pipeline length must divide I")
    if new_k == old_k:
        return []
    fan = old_k // new_k
    return [(s, s + new_k * j) for s in active_ranks(nodes, gpn, old_k) for j in range(1, fan)]


def redistribute(dataset: int, nodes: int, gpn: int, K: int, epoch: int, seed: int):
    """autodp.cpp:113-151 -> (ranks, shards)."""
    ranks = active_ranks(nodes, gpn, K)
    if dataset < len(ranks):
        raise ValueError("redistribute: dataset smaller than replica count")
    shards: List[List[int]] = [[] for _ in ranks]
    for n in range(nodes):
        subset = list(range(n, dataset, nodes))
        rng = SplitMix64(hash_combine(hash_combine(seed, epoch), n))
        deterministic_shuffle(subset, rng)
        slots = [s for s, r in enumerate(ranks) if r // gpn == n]
        per, extra = divmod(len(subset), len(slots))
        cur = 0
        for j, s in enumerate(slots):
            ln = per + (1 if j < extra else 0)
            shards[s] = subset[cur:cur + ln]
            cur += ln
    return ranks, shards


# ---- autocache.cpp -------------------------------------------------------------
@dataclass
class Tiers:
    host_bandwidth: float = 3.05e9
    disk_bandwidth: float = 6.0e9
    host_capacity_bytes: float = 64e9
    window_batches: int = 64
    block_batches: int = 8
    read_latency: float = 0.0


def cache_read_s(m: Model, boundary: int, t: Tiers) -> float:  # autocache.cpp:23-29
    if boundary <= 0:
        return 0.0
    return float(m.act[2 * boundary]) / t.host_bandwidth + t.read_latency


def should_cache(lf: int, m: Model, cm: Cost, t: Tiers, mb: float) -> bool:
    """autocache.cpp:31-43."""
    read = cache_read_s(m, lf, t) * mb
    fwd = cm.c_fwd * float(m.prefix(lf)) * mb
    return lf > 0 and read < fwd


# ---- runner.cpp: decision trajectory -------------------------------------------
def trajectory(cfg: dict, model: Model, norms_fn=None) -> List[Tuple[int, int, int, int, bool]]:
    """Decision order of simulate_run (runner.cpp:94-229) -> per epoch
    (L_frozen, K, R, M, cache_enabled).  `cfg` is a schema-v1 scenario dict
    (all features on, synthetic norms unless norms_fn is given)."""
    cl = cfg.get("cluster", {})
    nodes, gpn = cl.get("nodes", 1), cl.get("gpus_per_node", 1)
    cluster = dict(nodes=nodes, intra=cl.get("intra_node_bandwidth", 15.754e9),
                   inter=cl.get("inter_node_bandwidth", 5e9))
    tr = cfg.get("training", {})
    batch = float(tr.get("per_pipeline_batch", 400.0))
    epochs = tr.get("epochs", 10)
    ipe = tr.get("iterations_per_epoch", 100)
    alpha = tr.get("alpha", 1.0 / 3.0)
    lam = tr.get("lambda_frozen", 1.0 / 6.0)
    interval = tr.get("freeze_check_interval", 1)
    c = cfg.get("cost_model", {})
    cm = Cost(**{k: v for k, v in c.items() if k != "transition_overheads"})
    ca = cfg.get("cache", {})
    policy = ca.get("policy", "auto")
    tiers = Tiers(**{k: v for k, v in ca.items() if k != "policy"})
    feats = dict(freeze=True, autopipe=True, autodp=True, autocache=True)
    feats.update(cfg.get("features", {}))
    crit = 1 if cfg.get("balance_criterion") == "paper-variance" else 0
    gn = cfg.get("grad_norms", {})
    seed = cfg.get("seed", 1)
    gseed = gn.get("seed", 0) or seed
    profile = 1 if gn.get("profile") == "early-random" else 0
    switch = gn.get("switchover_epoch", 2)
    if norms_fn is None:
        def norms_fn(e):
            return synthetic_norms(profile, gseed, model.L, switch, e)

    k0 = cfg.get("initial_pipeline_length", 0) or gpn
    r0 = nodes * (gpn // k0)
    seq = m_partition(model, 0)
    plan = load_balance(seq, k0, lam, crit)
    micro, _ = optimal_chunks(plan, model, seq, batch, r0, cluster, cm)
    m_gpu0 = plan.max_eff()
    st = FreezeState(alpha)
    k, lf = k0, 0
    cache_on, boundary = False, 0
    out = []
    for epoch in range(epochs):
        changed = False
        if feats["freeze"] and epoch > 0 and epoch % interval == 0:
            nxt = next_frozen_count(st, norms_fn(epoch - 1), model.L)
            if nxt != lf:
                lf, changed = nxt, True
                seq = m_partition(model, lf)
                if feats["autopipe"]:
                    while k > 1 and len(seq.params) < k:
                        k //= 2
                    k, plan, _ = try_compress(seq, k, lam, m_gpu0, crit)
        R = nodes * (gpn // k) if feats["autodp"] else r0
        if (feats["autopipe"] and feats["autocache"] and policy != "always_off" and lf > 0):
            want = policy == "always_on" or should_cache(lf, model, cm, tiers, batch / micro)
            if want and (not cache_on or boundary < lf):
                cache_on, boundary = True, lf
        read = cache_read_s(model, boundary, tiers) if cache_on else 0.0
        if feats["autopipe"] and changed:
            micro, _ = optimal_chunks(plan, model, seq, batch, R, cluster, cm, cache_on, read)
        out.append((lf, k if feats["autopipe"] else k0, R, micro, cache_on))
    _ = ipe
    return out
