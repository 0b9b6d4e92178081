"""Seeded synthetic traces shaped like the paper's workloads.

Sources for every parameter (PAPER.md line numbers):

* Fig. 2 worked example: A{4,3,1,1}, B{3,3,4}, C{1,2}, D{4}, all chains,
  all arriving at t=0.
* ShareGPT (chatbot) P:L326: 6.66 calls/program (max 80), 256 prefill / 277
  decode tokens per call.
* BFCL (ReAct) P:L334: 10.75 calls/program (max 70), 735.06 prefill / 34.14 decode.
* LATS (MCTS) P:L336: 159.7 calls/program = MCTS iterations x (5 expand + 5 evaluate),
  467.2 prefill / 72.6 decode.
* Map-reduce, Fig. 1c: F parallel map calls joined by one reduce call.

Long-tailed quantities are log-normal, rounded and clipped to [1, max]; the (mu, sigma)
pairs are the fits recorded in SURVEY.md §8(d) (mean = paper mean, p99.9 = max).  The
RNG is NumPy's counter-based Philox, seeded with BASE_SEED + config index.

A trace is static workload description only: DAG edges, hidden decode lengths,
interrupt delays, token contexts and arrival steps.  What a scheduler does with it is
not in this package.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

BASE_SEED = 20250219
# config index per BASELINE.json "configs" order
CONFIG_INDEX = {"fig2": 0, "chatbot": 1, "react": 2, "mcts": 3, "multi": 4}

# (mu, sigma, max) per quantity, SURVEY.md §8(d) table
SHAREGPT_CALLS = (1.4442, 0.9507, 80)
SHAREGPT_DECODE = (5.0726, 1.0501, 4096)
SHAREGPT_PREFILL = (4.9521, 1.0891, 4096)
BFCL_CALLS = (2.1427, 0.6814, 70)
BFCL_DECODE = (2.5042, 1.4327, 1024)
BFCL_PREFILL = (6.1805, 0.9159, 8192)
LATS_ITERS = (2.6055, 0.5749, 80)
LATS_DECODE = (3.7575, 1.0271, 1024)
LATS_PREFILL = (5.8201, 0.8082, 4096)
MCTS_WIDTH = 5

# interrupt delays (assumed; the paper gives none): log-normal with these means, in steps
HUMAN_DELAY_MEAN = 50.0
TOOL_DELAY_MEAN = 200.0
DELAY_SIGMA = 1.0
MAX_CONTEXT = 32768


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def lognormal_clipped(rng, mu, sigma, vmax, size, vmin=1):
    x = np.rint(np.exp(rng.normal(mu, sigma, size)))
    return np.clip(x, vmin, vmax).astype(np.int64)


def _delays(rng, mean, size):
    mu = np.log(mean) - DELAY_SIGMA ** 2 / 2
    return lognormal_clipped(rng, mu, DELAY_SIGMA, 20 * mean, size, vmin=0)


@dataclass
class Trace:
    """Columnar program/call description.

    Calls of program p are the contiguous range first_call[p]:first_call[p+1], listed
    in a topological order (parents before children).  `par` holds global call indices;
    the parents of call c are par[par_ptr[c]:par_ptr[c+1]].
    """
    name: str
    prog_id: np.ndarray        # u64 [P]
    prog_arrival: np.ndarray   # i64 [P] arrival step of the program (its roots)
    first_call: np.ndarray     # i64 [P+1]
    call_prog: np.ndarray      # i64 [C] program index
    call_idx: np.ndarray       # i64 [C] index within the program
    call_id: np.ndarray        # u64 [C] = (program index << 16) | call index
    decode: np.ndarray         # i64 [C] hidden decode length (engine steps), >= 1
    prefill: np.ndarray        # i64 [C] the call's own new prompt tokens
    input_tokens: np.ndarray   # i64 [C] full input context of the call (drives KV blocks, Alg. 2 LEN)
    delay: np.ndarray          # i64 [C] interrupt delay between parents' completion and arrival
    par_ptr: np.ndarray        # i64 [C+1]
    par: np.ndarray            # i64 [E]
    meta: dict = field(default_factory=dict)

    @property
    def n_programs(self):
        return len(self.prog_id)

    @property
    def n_calls(self):
        return len(self.call_id)

    def parents(self, c):
        return self.par[self.par_ptr[c]:self.par_ptr[c + 1]]

    def children_csr(self):
        """Reverse adjacency (child lists) as CSR: (ptr[C+1], child[E])."""
        C = self.n_calls
        cnt = np.bincount(self.par, minlength=C) if len(self.par) else np.zeros(C, np.int64)
        ptr = np.zeros(C + 1, np.int64)
        np.cumsum(cnt, out=ptr[1:])
        child_of_edge = np.repeat(np.arange(C), np.diff(self.par_ptr))
        order = np.argsort(self.par, kind="stable")
        return ptr, child_of_edge[order]

    def validate(self):
        C = self.n_calls
        assert np.all(self.decode >= 1), "decode_tokens must be >= 1"
        assert self.first_call[0] == 0 and self.first_call[-1] == C
        for c in range(C) if C < 5000 else []:
            for p in self.parents(c):
                assert p < c and self.call_prog[p] == self.call_prog[c], "parent must precede, same program"
        return True


def _assemble(name, progs, arrivals, prog_ids=None, meta=None):
    """progs: list of dicts with decode, prefill, delay (arrays) and parents (list of
    lists of local indices), input_tokens (array).  Builds the columnar Trace."""
    P = len(progs)
    sizes = np.array([len(p["decode"]) for p in progs], np.int64)
    first = np.zeros(P + 1, np.int64)
    np.cumsum(sizes, out=first[1:])
    C = int(first[-1])
    call_prog = np.repeat(np.arange(P, dtype=np.int64), sizes)
    call_idx = np.arange(C, dtype=np.int64) - first[call_prog]
    assert sizes.max(initial=0) < (1 << 16)
    if prog_ids is None:
        prog_ids = np.arange(P, dtype=np.uint64)
    call_id = (call_prog.astype(np.uint64) << np.uint64(16)) | call_idx.astype(np.uint64)
    cat = lambda k: np.concatenate([np.asarray(p[k], np.int64) for p in progs]) if P else np.zeros(0, np.int64)
    par_counts, par_list = [], []
    for pi, p in enumerate(progs):
        base = first[pi]
        for plist in p["parents"]:
            par_counts.append(len(plist))
            par_list.extend(int(base + x) for x in plist)
    par_ptr = np.zeros(C + 1, np.int64)
    np.cumsum(np.array(par_counts, np.int64), out=par_ptr[1:])
    return Trace(name=name, prog_id=np.asarray(prog_ids, np.uint64),
                 prog_arrival=np.asarray(arrivals, np.int64), first_call=first,
                 call_prog=call_prog, call_idx=call_idx, call_id=call_id,
                 decode=cat("decode"), prefill=cat("prefill"),
                 input_tokens=np.minimum(cat("input_tokens"), MAX_CONTEXT),
                 delay=cat("delay"), par_ptr=par_ptr, par=np.array(par_list, np.int64),
                 meta=meta or {})


def _chain(decode, prefill, delay, system_prompt=0):
    decode = np.asarray(decode, np.int64)
    prefill = np.asarray(prefill, np.int64)
    n = len(decode)
    # cumulative context: system prompt + all earlier prefill/decode + own prefill
    ctx = system_prompt + np.cumsum(prefill) + np.concatenate([[0], np.cumsum(decode)[:-1]])
    return dict(decode=decode, prefill=prefill, delay=np.asarray(delay, np.int64),
                parents=[[] if i == 0 else [i - 1] for i in range(n)], input_tokens=ctx)


def _dag_ctx(decode, prefill, parents, system_prompt=0):
    ctx = np.zeros(len(decode), np.int64)
    for i, ps in enumerate(parents):
        up = max((ctx[p] + decode[p] for p in ps), default=system_prompt)
        ctx[i] = up + prefill[i]
    return ctx


def dag_trace(name, programs, arrivals) -> Trace:
    """A trace from explicit per-program lists: each program is a dict with decode, parents
    (local indices) and optionally delay / prefill (default 0 / 1)."""
    progs = []
    for p in programs:
        n = len(p["decode"])
        dec = np.asarray(p["decode"], np.int64)
        pre = np.asarray(p.get("prefill", [1] * n), np.int64)
        progs.append(dict(decode=dec, prefill=pre, delay=np.asarray(p.get("delay", [0] * n), np.int64),
                          parents=p["parents"], input_tokens=_dag_ctx(dec, pre, p["parents"])))
    return _assemble(name, progs, arrivals)


def fig2() -> Trace:
    """Fig. 2a: decode steps per LLM call, BS=2, all programs at t=0."""
    dec = {"A": [4, 3, 1, 1], "B": [3, 3, 4], "C": [1, 2], "D": [4]}
    progs = [_chain(d, [1] * len(d), [0] * len(d)) for d in dec.values()]
    return _assemble("fig2", progs, [0, 0, 0, 0], meta={"names": list(dec)})


def atlas_dag_fixture() -> Trace:
    """Derived ATLAS-vs-PLAS regression DAG (SURVEY.md §8(c) 'What pins each part';
    not from the paper).  P0: c0(2) -> {c1(3), c2(3)}, c1 -> c3(2).
    P1: c0(2) -> c1(1); {c0, c1} -> c2(3), c3(3)."""
    p0 = dict(decode=[2, 3, 3, 2], parents=[[], [0], [0], [1]])
    p1 = dict(decode=[2, 1, 3, 3], parents=[[], [0], [0, 1], [0, 1]])
    progs = []
    for p in (p0, p1):
        n = len(p["decode"])
        pre = np.ones(n, np.int64)
        progs.append(dict(decode=np.array(p["decode"]), prefill=pre, delay=np.zeros(n, np.int64),
                          parents=p["parents"],
                          input_tokens=_dag_ctx(np.array(p["decode"]), pre, p["parents"])))
    return _assemble("atlas_dag", progs, [0, 0])


def random_tiny(seed: int, max_programs=4, max_calls=4, max_decode=4, max_delay=2,
                max_arrival=3, dag=True, max_prefill=6) -> Trace:
    """Tiny random traces for brute-force / property tests: chains and 2-parent DAGs."""
    rng = rng_for(BASE_SEED * 7919 + seed)
    P = int(rng.integers(1, max_programs + 1))
    progs, arr = [], []
    for _ in range(P):
        n = int(rng.integers(1, max_calls + 1))
        parents = []
        for i in range(n):
            if i == 0:
                parents.append([])
            elif dag and i >= 2 and rng.random() < 0.4:
                a, b = rng.choice(i, size=2, replace=False)
                parents.append(sorted([int(a), int(b)]))
            elif dag and rng.random() < 0.3:
                parents.append([int(rng.integers(0, i))])
            else:
                parents.append([i - 1])
        dec = rng.integers(1, max_decode + 1, n)
        pre = rng.integers(0, max_prefill + 1, n)
        dl = rng.integers(0, max_delay + 1, n)
        dl[0] = 0
        progs.append(dict(decode=dec, prefill=pre, delay=dl, parents=parents,
                          input_tokens=_dag_ctx(dec, pre, parents)))
        arr.append(int(rng.integers(0, max_arrival + 1)))
    return _assemble(f"tiny{seed}", progs, arr)


def _poisson_arrivals(rng, n, rate):
    if rate is None:
        return np.zeros(n, np.int64)  # offline burst
    return np.floor(np.cumsum(rng.exponential(1.0 / rate, n))).astype(np.int64)


def chatbot(n_programs=10_000, seed=None, rate=None, system_prompt=0) -> Trace:
    """ShareGPT-shaped chains with human-turn interrupts."""
    rng = rng_for(BASE_SEED + CONFIG_INDEX["chatbot"] if seed is None else seed)
    ncalls = lognormal_clipped(rng, *SHAREGPT_CALLS, n_programs)
    C = int(ncalls.sum())
    dec = lognormal_clipped(rng, *SHAREGPT_DECODE, C)
    pre = lognormal_clipped(rng, *SHAREGPT_PREFILL, C)
    dl = _delays(rng, HUMAN_DELAY_MEAN, C)
    arr = _poisson_arrivals(rng, n_programs, rate)
    return _chains_trace("chatbot", ncalls, dec, pre, dl, arr, system_prompt)


def react(n_programs=10_000, seed=None, rate=None, system_prompt=0) -> Trace:
    """BFCL-shaped ReAct chains with tool interrupts."""
    rng = rng_for(BASE_SEED + CONFIG_INDEX["react"] if seed is None else seed)
    ncalls = lognormal_clipped(rng, *BFCL_CALLS, n_programs)
    C = int(ncalls.sum())
    dec = lognormal_clipped(rng, *BFCL_DECODE, C)
    pre = lognormal_clipped(rng, *BFCL_PREFILL, C)
    dl = _delays(rng, TOOL_DELAY_MEAN, C)
    arr = _poisson_arrivals(rng, n_programs, rate)
    return _chains_trace("react", ncalls, dec, pre, dl, arr, system_prompt)


def _chains_trace(name, ncalls, dec, pre, dl, arr, system_prompt):
    """Vectorised chain assembly (same result as _chain per program)."""
    P = len(ncalls)
    first = np.zeros(P + 1, np.int64)
    np.cumsum(ncalls, out=first[1:])
    C = int(first[-1])
    call_prog = np.repeat(np.arange(P, dtype=np.int64), ncalls)
    call_idx = np.arange(C, dtype=np.int64) - first[call_prog]
    dl = dl.copy()
    dl[call_idx == 0] = 0
    # ctx = system + cumsum(prefill) within program + cumsum(decode) of earlier calls
    cpre = np.cumsum(pre)
    cdec = np.cumsum(dec)
    base_pre = np.concatenate([[0], cpre])[first[call_prog]]
    base_dec = np.concatenate([[0], cdec])[first[call_prog]]
    ctx = system_prompt + (cpre - base_pre) + (cdec - dec - base_dec)
    has_par = call_idx > 0
    par_ptr = np.zeros(C + 1, np.int64)
    np.cumsum(has_par.astype(np.int64), out=par_ptr[1:])
    par = np.nonzero(has_par)[0] - 1
    call_id = (call_prog.astype(np.uint64) << np.uint64(16)) | call_idx.astype(np.uint64)
    return Trace(name=name, prog_id=np.arange(P, dtype=np.uint64), prog_arrival=arr,
                 first_call=first, call_prog=call_prog, call_idx=call_idx, call_id=call_id,
                 decode=dec, prefill=pre, input_tokens=np.minimum(ctx, MAX_CONTEXT), delay=dl,
                 par_ptr=par_ptr, par=par.astype(np.int64))


def _mcts_program(rng, iters, w=MCTS_WIDTH):
    """Round r: expand E_{r,1..w}, each depending on ALL evaluates of round r-1 (the
    join; roots when r=1); then evaluate V_{r,i} depending on E_{r,i}.  10*I calls."""
    n = 2 * w * iters
    dec = lognormal_clipped(rng, *LATS_DECODE, n)
    pre = lognormal_clipped(rng, *LATS_PREFILL, n)
    parents = []
    prev_v = []
    for r in range(iters):
        base = 2 * w * r
        for i in range(w):
            parents.append(list(prev_v))
        for i in range(w):
            parents.append([base + i])
        prev_v = [base + w + i for i in range(w)]
    return dict(decode=dec, prefill=pre, delay=np.zeros(n, np.int64), parents=parents,
                input_tokens=_dag_ctx(dec, pre, parents))


def _mapreduce_program(rng, fan):
    n = fan + 1
    dec = lognormal_clipped(rng, *LATS_DECODE, n)
    pre = lognormal_clipped(rng, *LATS_PREFILL, n)
    parents = [[] for _ in range(fan)] + [list(range(fan))]
    return dict(decode=dec, prefill=pre, delay=np.zeros(n, np.int64), parents=parents,
                input_tokens=_dag_ctx(dec, pre, parents))


def mcts_mapreduce(n_programs=28_000, seed=None, rate=None, frac_mcts=0.5) -> Trace:
    """50/50 LATS-MCTS and map-reduce DAG programs, vectorised.

    MCTS program with I iterations: calls 10r+i (i<5) are the expands E_{r,i}, each depending
    on all evaluates of round r-1 (roots when r=0); calls 10r+5+i are the evaluates V_{r,i},
    depending on E_{r,i} (same structure as `_mcts_program`).  Map-reduce program: F root maps,
    then one reduce depending on all of them (`_mapreduce_program`)."""
    rng = rng_for(BASE_SEED + CONFIG_INDEX["mcts"] if seed is None else seed)
    n = n_programs
    kinds = rng.random(n) < frac_mcts
    iters = lognormal_clipped(rng, *LATS_ITERS, n)
    fans = rng.integers(8, 129, n).astype(np.int64)
    sizes = np.where(kinds, 2 * MCTS_WIDTH * iters, fans + 1).astype(np.int64)
    first = np.zeros(n + 1, np.int64)
    np.cumsum(sizes, out=first[1:])
    C = int(first[-1])
    call_prog = np.repeat(np.arange(n, dtype=np.int64), sizes)
    local = np.arange(C, dtype=np.int64) - first[call_prog]
    dec = lognormal_clipped(rng, *LATS_DECODE, C)
    pre = lognormal_clipped(rng, *LATS_PREFILL, C)
    is_m = kinds[call_prog]
    W = MCTS_WIDTH
    r = local // (2 * W)
    k = local % (2 * W)
    mE = is_m & (k < W) & (r >= 1)
    mV = is_m & (k >= W)
    mR = (~is_m) & (local == fans[call_prog])
    cnt = np.zeros(C, np.int64)
    cnt[mE] = W
    cnt[mV] = 1
    cnt[mR] = fans[call_prog[mR]]
    par_ptr = np.zeros(C + 1, np.int64)
    np.cumsum(cnt, out=par_ptr[1:])
    par = np.empty(int(par_ptr[-1]), np.int64)
    cE = np.nonzero(mE)[0]
    baseE = first[call_prog[cE]] + 2 * W * (r[cE] - 1) + W          # V_{r-1,0}
    par[(par_ptr[cE][:, None] + np.arange(W)).ravel()] = (baseE[:, None] + np.arange(W)).ravel()
    cV = np.nonzero(mV)[0]
    par[par_ptr[cV]] = cV - W                                        # E_{r,i}
    cR = np.nonzero(mR)[0]
    F = fans[call_prog[cR]]
    pos = np.repeat(par_ptr[cR], F) + (np.arange(int(F.sum())) - np.repeat(np.cumsum(F) - F, F))
    par[pos] = np.repeat(first[call_prog[cR]], F) + (pos - np.repeat(par_ptr[cR], F))
    # contexts along the longest-token ancestor chain
    ctx = pre.copy()
    if len(cR):
        mp = np.nonzero(~kinds)[0]
        starts = first[mp]
        best = _segmax(ctx + dec, starts, fans[mp])   # over the F maps of each program
        ctx[first[mp] + fans[mp]] = pre[first[mp] + fans[mp]] + best
    mps = np.nonzero(kinds)[0]
    I = iters[mps]
    for rr in range(int(I.max()) if len(I) else 0):
        act = mps[I > rr]
        E = (first[act] + 2 * W * rr)[:, None] + np.arange(W)
        V = E + W
        if rr > 0:
            Vp = V - 2 * W
            ctx[E] = pre[E] + (ctx[Vp] + dec[Vp]).max(axis=1)[:, None]
        ctx[V] = pre[V] + ctx[E] + dec[E]
    call_id = (call_prog.astype(np.uint64) << np.uint64(16)) | local.astype(np.uint64)
    arr = _poisson_arrivals(rng, n, rate)
    t = Trace(name="mcts_mapreduce", prog_id=np.arange(n, dtype=np.uint64), prog_arrival=arr,
              first_call=first, call_prog=call_prog, call_idx=local, call_id=call_id, decode=dec,
              prefill=pre, input_tokens=np.minimum(ctx, MAX_CONTEXT), delay=np.zeros(C, np.int64),
              par_ptr=par_ptr, par=par)
    t.meta["is_mcts"] = kinds
    return t


def _segmax(x, starts, lens):
    """max of x[s:s+l] for each (s, l), vectorised."""
    idx = np.repeat(starts, lens) + (np.arange(int(lens.sum())) - np.repeat(np.cumsum(lens) - lens, lens))
    seg = np.repeat(np.arange(len(starts)), lens)
    out = np.full(len(starts), np.iinfo(np.int64).min)
    np.maximum.at(out, seg, x[idx])
    return out


def burst_mcts_mapreduce(target_active=1_000_000, seed=None) -> Trace:
    """Offline burst sized so that ~target_active calls are ready at step 0:
    each MCTS program contributes w=5 roots, each map-reduce program F ~ U{8..128}
    roots (mean 68), so ~36.5 roots per program on average."""
    n_prog = int(round(target_active / (0.5 * MCTS_WIDTH + 0.5 * 68)))
    return mcts_mapreduce(n_programs=n_prog, seed=seed)


def burst_mixed(target_active=4_000_000, seed=None) -> Trace:
    """BASELINE configs[4] on one engine: an offline burst of an equal draw of
    ShareGPT chat, BFCL ReAct and LATS MCTS / map-reduce programs.  n programs of each
    kind put about n + n + 36.5 n calls in the ready set at step 0 (a chain's first call; an MCTS
    program's w=5 roots, a map-reduce program's F ~ U{8..128} maps)."""
    rng = rng_for(BASE_SEED + CONFIG_INDEX["multi"] if seed is None else seed)
    n = int(round(target_active / (2 + 0.5 * MCTS_WIDTH + 0.5 * 68)))
    s = [int(x) for x in rng.integers(0, 1 << 30, 3)]
    return concat([chatbot(n, seed=s[0]), react(n, seed=s[1]), mcts_mapreduce(n, seed=s[2])], name="mixed_burst")


def churn(n_programs=1_000_000, calls_per_program=4, seed=None) -> Trace:
    """Stress shape for the step's prologue (SURVEY §8(d) timing protocol step 2): chains of
    one-token calls with no interrupts, all submitted at step 0, so every call in a batch
    completes after one step and its successor arrives in the next: about BS completions and BS
    arrivals per step.  Prefills follow BFCL."""
    rng = rng_for(BASE_SEED + 100 if seed is None else seed)
    ncalls = np.full(n_programs, calls_per_program, np.int64)
    C = int(ncalls.sum())
    dec = np.ones(C, np.int64)
    pre = lognormal_clipped(rng, *BFCL_PREFILL, C)
    return _chains_trace("churn", ncalls, dec, pre, np.zeros(C, np.int64), np.zeros(n_programs, np.int64), 0)


def mixed(n_programs=30_000, seed=None, rate=None) -> Trace:
    """Equal draw from ShareGPT / BFCL / LATS-style programs."""
    rng = rng_for(BASE_SEED + CONFIG_INDEX["multi"] if seed is None else seed)
    kind = rng.integers(0, 3, n_programs)
    parts = []
    for k, fn in enumerate((chatbot, react, mcts_mapreduce)):
        m = int((kind == k).sum())
        parts.append(fn(m, seed=int(rng.integers(1 << 30))))
    progs = []
    for tr in parts:
        for p in range(tr.n_programs):
            a, b = tr.first_call[p], tr.first_call[p + 1]
            loc = [[int(x - a) for x in tr.parents(c)] for c in range(a, b)]
            progs.append(dict(decode=tr.decode[a:b], prefill=tr.prefill[a:b], delay=tr.delay[a:b],
                              parents=loc, input_tokens=tr.input_tokens[a:b]))
    arr = _poisson_arrivals(rng, len(progs), rate)
    return _assemble("mixed", progs, arr)


def concat(traces, name=None) -> Trace:
    """Concatenates traces (e.g. one generated shard per engine) into one workload; program
    indices, program ids and call ids are renumbered so they stay unique."""
    P = np.cumsum([0] + [t.n_programs for t in traces])
    C = np.cumsum([0] + [t.n_calls for t in traces])
    cat = lambda f: np.concatenate([getattr(t, f) for t in traces])
    call_prog = np.concatenate([t.call_prog + P[i] for i, t in enumerate(traces)])
    call_idx = cat("call_idx")
    first = np.concatenate([t.first_call[:-1] + C[i] for i, t in enumerate(traces)] + [[C[-1]]])
    par_ptr = np.concatenate([t.par_ptr[:-1] + sum(len(x.par) for x in traces[:i]) for i, t in enumerate(traces)]
                             + [[sum(len(x.par) for x in traces)]])
    par = np.concatenate([t.par + C[i] for i, t in enumerate(traces)])
    call_id = (call_prog.astype(np.uint64) << np.uint64(16)) | call_idx.astype(np.uint64)
    return Trace(name=name or "+".join(t.name for t in traces), prog_id=np.arange(P[-1], dtype=np.uint64),
                 prog_arrival=cat("prog_arrival"), first_call=first.astype(np.int64), call_prog=call_prog,
                 call_idx=call_idx, call_id=call_id, decode=cat("decode"), prefill=cat("prefill"),
                 input_tokens=cat("input_tokens"), delay=cat("delay"), par_ptr=par_ptr.astype(np.int64),
                 par=par.astype(np.int64))
