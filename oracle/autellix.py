"""CPU oracle of Autellix's program-aware scheduler (arXiv 2502.13965).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.
The product path (`paper_2502_13965_b200/`) never imports it and shares no code
with it; both sides consume traces from `autx_workload` (input generation only).

This is a plain, slow, step-by-step discrete-event simulation in exact integer
arithmetic, written from PAPER.md (citations `P:L<line>`), Alg. 1,
Alg. 2 and the readings of SURVEY.md §8(c) / DESIGN.md §3.  Per
engine step t (time unit = one decode iteration, reading R17):

  1. completions of step t-1 update the process table          Alg.1 l.1-7, l.16-18
        PLAS (and FCFS/MLFQ): svc[p] += exec(c)                   Eq. 1
        ATLAS:                svc[p] = max(svc[p], inh(c)+exec(c)) Alg.1 l.4
        all:                  pwait[p] += totwait(c)              Alg.1 l.5-6, reading R5
  2. arrivals at step t, canonical order, inherit svc[p]        Alg.1 l.9-14
        ATLAS_EQ2 (exact Eq. 2): inherit max over the call's
        parents of (p(parent) + t_parent), 0 for a root            reading R31
        q = min{i : inh < hi_i} (PLAS/ATLAS) or 0 (FCFS/MLFQ)   P:L253, reading R1
        quanta = Q[q]                                            Alg.1 l.13
  3. demotion: quanta <= 0 -> q = min(q+1, K-1), quanta = Q[q]  Alg.1 l.20-23
  4. anti-starvation: (pwait[p]+wait)/(svc[p]+mtime) >= beta     Alg.1 l.24-30
        (integer cross-multiplication; 0/0 never promotes)       readings R3, R4, R7
        -> q = 0, quanta = Q[0], wait = mtime = 0
  5. order by key (q, call arrival step, not-running, seq)       P:L255, readings R11, R12
  6. cutoff: longest prefix with count <= BS and sum kvb <= P,   Alg.1 l.32-39 (`break`)
     stop at the first misfit                                    reading R13
        batch, admit = batch - resident, preempt = resident - batch, swap bytes
  7. account: batch exec++ mtime++ quanta-- running; others wait++ totwait++

Multi-step scheduling with over-provisioning (reading R32),
`Config.sched_every` = N, `Config.overprovision` = X (N = 1, X = 0 is the plain path above):
  * a scheduling point is the first step, every N-th step after the last scheduling point, and
    any step whose carried-over resident list is empty (idle engines do not wait for the window);
  * at a scheduling point steps 3-6 run as above, but the cutoff takes the longest prefix with
    count <= BS + X (and sum kvb <= P): the resident set R; the batch is its first BS calls and
    the other <= X calls are "standby" — their KV is put on the GPU (admitted) so that they join
    the batch at once when a batch call finishes before the next scheduling point;
  * between scheduling points (window steps) demotion, anti-starvation and ordering do not run
    (the scheduler runs "once every N decoding steps"): the carried resident list (batch, then
    standby, minus completed calls) is walked in order while sum kvb <= P (stop at the first
    misfit); its first BS calls run, the rest stay standby, and the calls after the misfit are
    evicted (KV growth of running calls: lazy eviction, lowest priority first).  Arrivals wait
    for the next scheduling point;
  * admit = R - resident before (swap-in when the call has run, else a fresh allocation);
    preempt = resident before - R, in the previous R order; a preempted call that never ran has
    no KV content, so it is freed without a swap-out; quanta keep counting down in window steps
    and the demotion they trigger waits for the next scheduling point.

Two independent formulations of steps 5-6 are provided and cross-checked:
  * `order_sorted`:  sort every active call by the unique key and take the prefix;
  * `order_queues`:  Alg. 1's literal walk over Q_1..Q_K (each queue a list in
     call-arrival order, running calls first within an equal-arrival group).

Parity status: pinned (see tests/test_oracle_*.py and DESIGN.md §3).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional
import numpy as np

INF = None  # infinite quantum / budget / beta marker

FCFS, MLFQ, PLAS, ATLAS = "fcfs", "mlfq", "plas", "atlas"
# Exact Eq. 2 ATLAS: a new call inherits max over its parents of
# (parent's priority + parent's execution time) instead of the program's scalar (reading R31)
ATLAS_EQ2 = "atlas_eq2"


@dataclass
class Config:
    policy: str = PLAS
    K: int = 1
    q_hi: tuple = ()                 # K-1 upper bounds (half-open [lo, hi)), reading R1
    quanta: tuple = (INF,)           # K quanta in steps; None = infinite
    beta: tuple = (1, 0)             # (num, den); den == 0 -> beta = infinity (never promote)
    max_batch: int = 2               # BS
    kv_budget: Optional[int] = None  # P in blocks; None = unbounded
    block_tokens: int = 16
    block_bytes: int = 0             # bytes of one logical KV block over all layers (swap ledger)
    token_threshold: int = 2048      # Alg. 2 line 2
    sched_every: int = 1             # N: the scheduler runs once every N steps (R32)
    overprovision: int = 0           # X: resident standby calls beyond BS (R32)

    def check(self):
        assert self.policy in (FCFS, MLFQ, PLAS, ATLAS, ATLAS_EQ2)
        assert 1 <= self.K <= 16 and len(self.q_hi) == self.K - 1 and len(self.quanta) == self.K
        assert list(self.q_hi) == sorted(self.q_hi)
        assert all(q is None or q >= 1 for q in self.quanta)
        assert self.max_batch >= 1
        assert self.sched_every >= 1 and self.overprovision >= 0
        return self


# Golden Fig. 2 configurations (reading R2)
def fig2_config(policy: str) -> Config:
    if policy == FCFS:
        return Config(policy=FCFS, K=1, q_hi=(), quanta=(INF,), max_batch=2).check()
    if policy == MLFQ:
        return Config(policy=MLFQ, K=3, q_hi=(0, 0), quanta=(1, 2, INF), max_batch=2).check()
    return Config(policy=policy, K=2, q_hi=(1,), quanta=(1, INF), max_batch=2).check()


def spec_ladder_config(policy=PLAS, max_batch=256, kv_budget=None, beta=(2, 1), block_bytes=0):
    """SPEC default ladder: K=8, hi_i = 2*4^(i-1), quanta = band widths."""
    hi = tuple(2 * 4 ** i for i in range(7))
    lo = (0,) + hi
    quanta = tuple(hi[i] - lo[i] for i in range(7)) + (INF,)
    return Config(policy=policy, K=8, q_hi=hi, quanta=quanta, beta=beta, max_batch=max_batch,
                  kv_budget=kv_budget, block_bytes=block_bytes).check()


class ProgramTable:
    """Global process table: one entry per program, keyed by program id."""

    def __init__(self):
        self.svc = {}        # service: PLAS sum / ATLAS longest critical path
        self.pwait = {}      # total waiting time of completed calls
        self.last_arrival = {}
        self.last_completion = {}

    def ensure(self, pid, t):
        if pid not in self.svc:
            self.svc[pid] = 0
            self.pwait[pid] = 0
            self.last_arrival[pid] = t
            self.last_completion[pid] = None

    def apply_completion(self, policy, pid, exec_steps, inh, totwait, t):
        """UPDATE_PROCESS_TABLE, Alg. 1 l.1-7."""
        if policy in (ATLAS, ATLAS_EQ2):
            self.svc[pid] = max(self.svc[pid], inh + exec_steps)  # Alg. 1 l.4 / Eq. 2 scalar
        else:
            self.svc[pid] = self.svc[pid] + exec_steps               # Eq. 1 sum
        self.pwait[pid] += totwait
        self.last_completion[pid] = t

    def end_program(self, pid):
        for d in (self.svc, self.pwait, self.last_arrival, self.last_completion):
            d.pop(pid, None)


@dataclass
class Call:
    cid: int
    pid: int
    arr: int            # call arrival step
    parr: int           # program arrival step (canonical order only)
    seq: int            # registration sequence number
    input_tokens: int
    inh: int            # service inherited at arrival (Alg. 1 l.11)
    q: int
    quanta: Optional[int]
    wait: int = 0       # c.wait, reset on promotion
    mtime: int = 0      # c.model_time, reset on promotion
    exec: int = 0       # t_k, never reset (reading R6)
    totwait: int = 0    # waiting steps since arrival, never reset (reading R5)
    running: bool = False   # in the previous step's batch
    resident: bool = False  # KV blocks on the GPU
    held: int = 0           # KV blocks held (on GPU if resident, on host otherwise)


class CapacityError(ValueError):
    """KV need of a single call exceeds the budget P (reading R14; AUTX_E_NOMEM)."""


def ceil_div(a, b):
    return -(-a // b)


class Engine:
    """One serving engine's scheduler state (Alg. 1) over a (possibly shared) table."""

    def __init__(self, cfg: Config, table: Optional[ProgramTable] = None, check_formulations=True):
        self.cfg = cfg.check()
        self.table = table if table is not None else ProgramTable()
        self.calls = {}          # cid -> Call (active calls)
        self.next_seq = 0
        self.prev_batch = []     # cids of the previous step's batch, in batch order
        self.standby = []        # R32: resident, not running (after the batch in R order)
        self.since = None        # R32: steps since the last scheduling point (None: none yet)
        self.check = check_formulations
        self.last_arrival_key = None
        self.crit = {}           # ATLAS_EQ2: completed cid -> p(c) + t_c (Eq. 2 operand)
        self.crit_of_prog = {}   # pid -> completed cids kept in self.crit

    # -- Alg. 1 helpers ------------------------------------------------------------
    def quantum(self, q):
        return self.cfg.quanta[q]

    def place(self, service):
        """Alg. 1 l.12: Q_i^lo <= service < Q_i^hi (half-open, reading R1)."""
        if self.cfg.policy in (FCFS, MLFQ):
            return 0
        for i, hi in enumerate(self.cfg.q_hi):
            if service < hi:
                return i
        return self.cfg.K - 1

    def kvb(self, c: Call):
        """Blocks needed to run the call's next token (reading R14)."""
        return ceil_div(c.input_tokens + c.exec + 1, self.cfg.block_tokens)

    def key(self, c: Call):
        return (c.q, c.arr, 0 if c.running else 1, c.seq)

    # -- step phases ---------------------------------------------------------------
    def complete(self, t, cids):
        """Phase 1 (local part): remove completed calls, return their table records."""
        recs = []
        for cid in sorted(cids, key=lambda x: self.calls[x].seq):
            c = self.calls[cid]
            if not c.running:
                raise ValueError(f"call {cid} completed but did not run in step {t-1}")
            recs.append((c.pid, c.exec, c.inh, c.totwait))
            if self.cfg.policy == ATLAS_EQ2:
                self.crit[cid] = c.inh + c.exec                   # p(c_k) + t_k, Eq. 2
                self.crit_of_prog.setdefault(c.pid, []).append(cid)
            del self.calls[cid]
        self.prev_batch = [x for x in self.prev_batch if x in self.calls]
        self.standby = [x for x in self.standby if x in self.calls]
        return recs

    def apply_records(self, t, recs):
        for pid, ex, inh, tw in recs:
            self.table.apply_completion(self.cfg.policy, pid, ex, inh, tw, t)

    def eq2_priority(self, pid, parents):
        """Eq. 2: 0 for a root, else max over the parents c_k of p(c_k) + t_k.  The
        parents must be completed calls of the same program ("parents P(c_j) in the same
        program")."""
        if not parents:
            return 0
        for k in parents:
            if k not in self.crit or k not in self.crit_of_prog.get(pid, ()):
                raise KeyError(f"parent {k} is not a completed call of program {pid}")
        return max(self.crit[k] for k in parents)

    def end_program(self, pid):
        """end_session: the table entry and the program's Eq. 2 operands go."""
        self.table.end_program(pid)
        for k in self.crit_of_prog.pop(pid, []):
            del self.crit[k]

    def register(self, t, arrivals, parents=None):
        """Phase 2: arrivals = list of (cid, pid, arrival_step, program_arrival_step,
        input_tokens) in canonical order: (arr, parr, pid, cid).  ATLAS_EQ2 also
        takes parents: cid -> list of parent cids."""
        for (cid, pid, arr, parr, tok) in arrivals:
            k = (arr, parr, pid, cid)
            if self.last_arrival_key is not None and k <= self.last_arrival_key:
                raise ValueError("arrivals not in canonical order")
            self.last_arrival_key = k
            if arr != t:
                raise ValueError("arrival step must equal the current step")
            if cid in self.calls:
                raise ValueError("duplicate call id")
            self.table.ensure(pid, t)
            self.table.last_arrival[pid] = t
            if self.cfg.policy == ATLAS_EQ2:
                inh = self.eq2_priority(pid, (parents or {}).get(cid, ()))   # Eq. 2
            else:
                inh = self.table.svc[pid]                   # Alg. 1 l.11
            q = self.place(inh)                              # Alg. 1 l.12
            c = Call(cid=cid, pid=pid, arr=arr, parr=parr, seq=self.next_seq, input_tokens=tok,
                     inh=inh, q=q, quanta=self.quantum(q))   # Alg. 1 l.13
            self.next_seq += 1
            if self.cfg.kv_budget is not None and self.kvb(c) > self.cfg.kv_budget:
                raise ValueError("initial kvb exceeds the KV budget (reading R13)")
            self.calls[cid] = c

    def demote_and_promote(self):
        """Phases 3-4 over every active call (reading R8), demotion first (R9)."""
        K = self.cfg.K
        num, den = self.cfg.beta
        for c in self.calls.values():
            if c.quanta is not None and c.quanta <= 0:               # Alg. 1 l.20-23
                c.q = min(c.q + 1, K - 1)
                c.quanta = self.quantum(c.q)
            W = self.table.pwait[c.pid] + c.wait                     # Alg. 1 l.24
            T = self.table.svc[c.pid] + c.mtime                      # Alg. 1 l.25
            if den != 0 and not (W == 0 and T == 0) and W * den >= num * T:  # l.26, R3/R4
                c.q = 0                                               # l.27
                c.quanta = self.quantum(0)                            # reading R7
                c.wait = 0                                            # l.29
                c.mtime = 0

    def fits(self, count, kv_sum, c):
        if count + 1 > self.cfg.max_batch + self.cfg.overprovision:   # R32: BS + X resident
            return False
        P = self.cfg.kv_budget
        return P is None or kv_sum + self.kvb(c) <= P

    def order_sorted(self):
        """Formulation (ii): sort by the unique key, take the feasible prefix."""
        order = sorted(self.calls.values(), key=self.key)
        batch, n, kv = [], 0, 0
        for c in order:
            if not self.fits(n, kv, c):
                break                                                   # Alg. 1 l.37
            batch.append(c.cid)
            n += 1
            kv += self.kvb(c)
        return batch

    def order_queues(self):
        """Formulation (i): Alg. 1 l.32-39 walk over Q_1..Q_K; each queue is a FIFO by
        call arrival (reading R11); inside one arrival step the call that ran in the
        previous step goes first (reading R12), then registration order."""
        queues = [[] for _ in range(self.cfg.K)]
        for c in sorted(self.calls.values(), key=lambda c: (c.arr, c.seq)):
            queues[c.q].append(c)
        batch, n, kv = [], 0, 0
        for Q in queues:
            i = 0
            while i < len(Q):
                j = i
                while j < len(Q) and Q[j].arr == Q[i].arr:
                    j += 1
                group = [c for c in Q[i:j] if c.running] + [c for c in Q[i:j] if not c.running]
                for c in group:
                    if not self.fits(n, kv, c):
                        return batch
                    batch.append(c.cid)
                    n += 1
                    kv += self.kvb(c)
                i = j
        return batch

    def schedule(self, t):
        """Phases 5-7; returns the decision record."""
        batch = self.order_sorted()
        if self.calls and not batch:
            # the head call alone needs more than P blocks: with Alg. 1's `break` nothing can
            # ever run again; reading R14 makes this a capacity error (AUTX_E_NOMEM)
            raise CapacityError(f"t={t}: a call's KV need exceeds the budget (reading R14)")
        if self.check:
            alt = self.order_queues()
            assert alt == batch, f"formulations disagree at t={t}: {batch} vs {alt}"
        return self._commit(t, batch)

    def window(self, t):
        """R32 window step: the carried resident list, walked in order under the KV budget."""
        res, n, kv = [], 0, 0
        for x in self.prev_batch + self.standby:
            c = self.calls[x]
            if not self.fits(n, kv, c):
                break                                                   # lazy eviction
            res.append(x)
            n += 1
            kv += self.kvb(c)
        if self.calls and not res:
            raise CapacityError(f"t={t}: a call's KV need exceeds the budget (reading R14)")
        return self._commit(t, res)

    def _commit(self, t, res):
        """Lists, swap ledger and step accounting (phases 6-7) for resident set `res` (in
        order): the first BS calls run, the rest are standby (R32; none when X = 0)."""
        BS = self.cfg.max_batch
        batch, standby = res[:BS], res[BS:]
        in_res, in_batch = set(res), set(batch)
        prev = self.prev_batch + self.standby
        admit = [x for x in res if not self.calls[x].resident]
        preempt = [x for x in prev if x not in in_res]
        bb = self.cfg.block_bytes
        # a call that never ran has no KV content: no host copy either way (R28, R32)
        swap_out = sum(self.calls[x].held for x in preempt if self.calls[x].exec > 0) * bb
        swap_in = sum(self.calls[x].held for x in admit if self.calls[x].exec > 0) * bb
        blocks = sum(self.kvb(self.calls[x]) for x in res)
        for x in preempt:
            self.calls[x].resident = False
        for x in res:
            self.calls[x].resident = True
        for c in self.calls.values():                                   # phase 7
            if c.cid in in_batch:
                c.exec += 1
                c.mtime += 1
                if c.quanta is not None:
                    c.quanta -= 1
                c.running = True
            else:
                c.wait += 1
                c.totwait += 1
                c.running = False
        for x in res:   # R28: a resident call holds the blocks of its KV, ceil((input + exec) / bt)
            c = self.calls[x]
            c.held = ceil_div(c.input_tokens + c.exec, self.cfg.block_tokens)
        self.prev_batch = list(batch)
        self.standby = list(standby)
        rec = dict(t=t, batch=batch, admit=admit, preempt=preempt, swap_out=swap_out,
                   swap_in=swap_in, kv_blocks=blocks, n_active=len(self.calls))
        if self.cfg.overprovision or self.cfg.sched_every > 1:
            rec["standby"] = standby
        return rec

    def sched_point(self):
        """R32: does this step run the scheduler (after completions and arrivals)?"""
        carried = self.prev_batch + self.standby
        return self.since is None or self.since >= self.cfg.sched_every or not carried

    def step(self, t, completed, arrivals, parents=None):
        recs = self.complete(t, completed)
        self.apply_records(t, recs)
        self.register(t, arrivals, parents)
        if self.sched_point():
            self.demote_and_promote()
            rec = self.schedule(t)
            self.since = 1
        else:
            rec = self.window(t)
            self.since += 1
        return rec

    def load(self):
        """Alg. 2 QUERY_ENGINE_WORKLOADS: queued + running calls (reading R21)."""
        return len(self.calls)


# ---------------------------------------------------------------------------------
# Alg. 2 load balancer
# ---------------------------------------------------------------------------------
def route(arrivals, loads, pins, threshold=2048):
    """Alg. 2 over a batch of arrivals in canonical order.

    arrivals: list of (cid, pid, input_tokens); loads: list of per-engine loads
    (mutated: +1 after each assignment, reading R23); pins: dict pid -> engine
    (mutated on the first long call, Alg. 2 l.10).  Ties -> lowest engine id.
    """
    if len(loads) == 0:
        raise ValueError("empty engine set")
    out = []
    for cid, pid, tok in arrivals:
        if tok <= threshold:                                   # l.2 small request
            e = min(range(len(loads)), key=lambda i: (loads[i], i))
        elif pid in pins:                                       # l.5-6
            e = pins[pid]
        else:                                                   # l.8-10
            e = min(range(len(loads)), key=lambda i: (loads[i], i))
            pins[pid] = e
        loads[e] += 1
        out.append(e)
    return out


def route_least_used(arrivals, loads):
    """The Least Used comparator of §6.4: every call to the engine with the fewest LLM
    calls in the system (ties -> lowest id), no pinning; loads +1 per assignment (R23)."""
    out = []
    for _ in arrivals:
        e = min(range(len(loads)), key=lambda i: (loads[i], i))
        loads[e] += 1
        out.append(e)
    return out


def route_round_robin(arrivals, n_engines, state):
    """The Round Robin comparator of §6.4: engines in cyclic order, one per call in
    canonical order; state = {"next": engine of the next call} persists across steps."""
    out = []
    for _ in arrivals:
        out.append(state["next"])
        state["next"] = (state["next"] + 1) % n_engines
    return out


ROUTERS = ("locality", "least_used", "round_robin")


class PrefixCache:
    """The program-prefix KV cache of the router's locality argument (§4.3; SPEC
    S:L183-191, reading R34): engine e holds, per program, the longest context (input + decoded
    tokens) of the program's calls it has served; a new call of the program there reuses at most
    its inherited context (its input tokens minus its own new prompt).  Prefill work = input
    tokens - reused tokens (a relative cost: the idealized engine's steps do not depend on it)."""

    def __init__(self, n_engines):
        self.ctx = [dict() for _ in range(n_engines)]
        self.prefill = 0
        self.hits = []   # (input tokens, reused tokens) per call

    def admit(self, e, pid, input_tokens, own_prefill):
        reused = min(self.ctx[e].get(pid, 0), input_tokens - own_prefill)
        self.prefill += input_tokens - reused
        self.hits.append((input_tokens, reused))
        return reused

    def done(self, e, pid, input_tokens, decode):
        self.ctx[e][pid] = max(self.ctx[e].get(pid, 0), input_tokens + decode)


# ---------------------------------------------------------------------------------
# Discrete-event harness: DAG readiness, hidden decode lengths, program end.
# ---------------------------------------------------------------------------------
class Workload:
    """Tracks readiness (parents done + interrupt delay elapsed) and the
    hidden decode lengths of a trace.  Not part of the scheduler (non-clairvoyance)."""

    def __init__(self, trace):
        self.tr = trace
        C = trace.n_calls
        self.n_par_left = np.diff(trace.par_ptr).astype(np.int64)
        self.ptr, self.child = trace.children_csr()
        self.ready_at = {}
        for c in np.nonzero(self.n_par_left == 0)[0]:
            p = trace.call_prog[c]
            self.ready_at.setdefault(int(trace.prog_arrival[p] + trace.delay[c]), []).append(int(c))
        self.remaining = trace.decode.astype(np.int64).copy()
        self.calls_left = np.diff(trace.first_call).astype(np.int64)
        self.done = 0
        self.index = {int(cid): i for i, cid in enumerate(trace.call_id)}
        self.finish = {}

    def arrivals(self, t):
        tr = self.tr
        cs = self.ready_at.pop(t, [])
        out = []
        for c in cs:
            p = tr.call_prog[c]
            out.append((int(tr.call_id[c]), int(tr.prog_id[p]), t, int(tr.prog_arrival[p]),
                        int(tr.input_tokens[c])))
        out.sort(key=lambda a: (a[2], a[3], a[1], a[0]))
        return out

    def ran(self, t, batch_cids):
        """Engine executed one decode step for each call in the batch at step t.
        Returns the completed call indices (processed at step t+1)."""
        done = []
        for cid in batch_cids:
            c = self.index[cid]
            self.remaining[c] -= 1
            if self.remaining[c] == 0:
                done.append(c)
        return done

    def release(self, t, done_idx):
        """Completions processed at step t release children at t + delay."""
        ended = []
        tr = self.tr
        for c in done_idx:
            self.done += 1
            p = int(tr.call_prog[c])
            self.calls_left[p] -= 1
            if self.calls_left[p] == 0:
                ended.append(int(tr.prog_id[p]))
                self.finish[int(tr.prog_id[p])] = t
            for ch in self.child[self.ptr[c]:self.ptr[c + 1]]:
                self.n_par_left[ch] -= 1
                if self.n_par_left[ch] == 0:
                    self.ready_at.setdefault(int(t + tr.delay[ch]), []).append(int(ch))
        return ended

    def finished(self):
        return self.done == self.tr.n_calls

    def parents_of(self, arrivals):
        """Parent call ids of each arrival (the DAG is the workload's; the scheduler
        learns a call's parents only when it arrives: non-clairvoyance)."""
        tr = self.tr
        out = {}
        for a in arrivals:
            c = self.index[a[0]]
            out[a[0]] = [int(tr.call_id[k]) for k in tr.parents(c)]
        return out


def simulate(trace, cfg: Config, max_steps=1_000_000, check_formulations=True, start=0):
    """Run a whole trace on one engine from step `start` (the trace's first arrival must not
    precede it); returns (log, metrics)."""
    eng = Engine(cfg, check_formulations=check_formulations)
    wl = Workload(trace)
    log = []
    completed = []
    total_wait = 0
    gantt = {}
    inh = {}
    for t in range(start, start + max_steps):
        if wl.finished():
            break
        done_cids = [int(trace.call_id[c]) for c in completed]
        for cid in done_cids:
            total_wait += eng.calls[cid].totwait
        ended = wl.release(t, completed)
        arr = wl.arrivals(t)
        rec = eng.step(t, done_cids, arr, wl.parents_of(arr) if cfg.policy == ATLAS_EQ2 else None)
        for a in arr:
            inh[a[0]] = eng.calls[a[0]].inh
        for pid in ended:
            eng.end_program(pid)
        log.append(rec)
        for cid in rec["batch"]:
            gantt.setdefault(cid, []).append(t)
        completed = wl.ran(t, rec["batch"])
    assert wl.finished(), "simulation did not finish"
    return log, dict(total_wait=total_wait, finish=dict(wl.finish), gantt=gantt, steps=len(log), inh=inh)


def gantt_strings(trace, gantt):
    """Per program: char at t = 1-based index of its call running at step t, else '.'."""
    out = {}
    for p in range(trace.n_programs):
        a, b = trace.first_call[p], trace.first_call[p + 1]
        steps = {}
        for c in range(a, b):
            for t in gantt.get(int(trace.call_id[c]), []):
                steps[t] = str(int(trace.call_idx[c]) + 1)
        end = max(steps) + 1 if steps else 0
        out[int(trace.prog_id[p])] = "".join(steps.get(t, ".") for t in range(end))
    return out


# ---------------------------------------------------------------------------------
# Multi-engine lockstep with a replicated process table (reading R22)
# ---------------------------------------------------------------------------------
def simulate_multi(trace, cfg: Config, n_engines: int, max_steps=1_000_000, router="locality", cache=None):
    """G engines step together.  Per step: local completions -> all completion
    records applied to the (replicated) table -> loads -> routing of the step's arrivals
    in canonical order (Alg. 2, or a §6.4 comparator) -> each engine schedules.
    cache: a PrefixCache that records each routed call's prefix reuse."""
    assert cfg.policy != ATLAS_EQ2, "Eq. 2 mode is single-engine (parents may run on other engines)"
    assert router in ROUTERS
    table = ProgramTable()
    engines = [Engine(cfg, table=table, check_formulations=False) for _ in range(n_engines)]
    wl = Workload(trace)
    pins = {}
    rr = {"next": 0}
    logs = [[] for _ in range(n_engines)]
    routes = []
    completed = [[] for _ in range(n_engines)]
    for t in range(max_steps):
        if wl.finished():
            break
        recs = []
        all_done = []
        for e, eng in enumerate(engines):
            cids = [int(trace.call_id[c]) for c in completed[e]]
            recs.extend(eng.complete(t, cids))
            all_done.extend(completed[e])
            if cache is not None:
                for c in completed[e]:
                    cache.done(e, int(trace.prog_id[trace.call_prog[c]]), int(trace.input_tokens[c]),
                               int(trace.decode[c]))
        for pid, ex, inh, tw in recs:
            table.apply_completion(cfg.policy, pid, ex, inh, tw, t)
        ended = wl.release(t, sorted(all_done))
        arr = wl.arrivals(t)
        loads = [eng.load() for eng in engines]
        if router == "locality":
            dest = route([(a[0], a[1], a[4]) for a in arr], loads, pins, cfg.token_threshold)
        elif router == "least_used":
            dest = route_least_used(arr, loads)
        else:
            dest = route_round_robin(arr, n_engines, rr)
        routes.append((t, [a[0] for a in arr], dest))
        if cache is not None:
            for a, e in zip(arr, dest):
                c = wl.index[a[0]]
                cache.admit(e, a[1], a[4], int(trace.prefill[c]))
        for e, eng in enumerate(engines):
            eng.register(t, [a for a, d in zip(arr, dest) if d == e])
        for e, eng in enumerate(engines):
            eng.demote_and_promote()
            rec = eng.schedule(t)
            logs[e].append(rec)
            completed[e] = wl.ran(t, rec["batch"])
        for pid in ended:
            table.end_program(pid)
            pins.pop(pid, None)
    return logs, routes
