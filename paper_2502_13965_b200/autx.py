"""Thin ctypes binding of libautx.so (include/autx.h).  Argument marshalling only: every step of
the scheduling path runs in the library's sm_100a kernels.  There is no fallback: if the shared
library or a GPU is missing, loading fails loudly."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libautx.so")

FCFS, MLFQ, PLAS, ATLAS = 0, 1, 2, 3
ATLAS_EQ2 = 4
POLICY = {"fcfs": FCFS, "mlfq": MLFQ, "plas": PLAS, "atlas": ATLAS, "atlas_eq2": ATLAS_EQ2}
ORDER_SELECT, ORDER_RADIX = 0, 1
ROUTE = {"locality": 0, "least_used": 1, "round_robin": 2}   # autx_route_policy
SWAP_SM, SWAP_PER_CHUNK_MEMCPY, SWAP_STAGED_DMA = 0, 1, 2
INF = 0xFFFFFFFF
STATUS = {0: "OK", 1: "E_INVAL", 2: "E_NOENT", 3: "E_EXIST", 4: "E_NOMEM", 5: "E_STATE",
          6: "E_CUDA", 7: "E_NCCL"}


class AutxError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Config(C.Structure):
    _fields_ = [("policy", C.c_int32), ("K", C.c_uint32), ("q_hi", C.c_uint32 * 15),
                ("quanta", C.c_uint32 * 16), ("beta_num", C.c_uint32), ("beta_den", C.c_uint32),
                ("max_batch", C.c_uint32), ("kv_budget_blocks", C.c_uint32),
                ("block_tokens", C.c_uint32), ("max_calls", C.c_uint32),
                ("max_programs", C.c_uint32), ("token_threshold", C.c_uint32),
                ("order_mode", C.c_uint32), ("n_gpu_blocks", C.c_uint32),
                ("max_blocks_per_call", C.c_uint32), ("host_pages", C.c_uint64),
                ("device", C.c_int32), ("stream", C.c_void_p), ("rank", C.c_int32),
                ("nranks", C.c_int32), ("route_policy", C.c_uint32), ("_reserved", C.c_uint32),
                ("nccl_comm", C.c_void_p), ("sched_every", C.c_uint32), ("overprovision", C.c_uint32)]


class StepOut(C.Structure):
    _fields_ = [("batch", C.c_void_p), ("admit", C.c_void_p), ("preempt", C.c_void_p),
                ("h_batch", C.POINTER(C.c_uint64)), ("h_admit", C.POINTER(C.c_uint64)),
                ("h_preempt", C.POINTER(C.c_uint64)), ("n_batch", C.c_uint32),
                ("n_admit", C.c_uint32), ("n_preempt", C.c_uint32), ("n_active", C.c_uint32),
                ("swap_out_blocks", C.c_uint64), ("swap_in_blocks", C.c_uint64),
                ("kv_blocks", C.c_uint64), ("n_promoted", C.c_uint32), ("n_standby", C.c_uint32),
                ("done", C.c_void_p)]


class KvLayout(C.Structure):
    _fields_ = [("k_pool", C.POINTER(C.c_void_p)), ("v_pool", C.POINTER(C.c_void_p)),
                ("n_layers", C.c_uint32), ("chunk_bytes", C.c_uint32),
                ("host_arena", C.c_void_p), ("host_arena_bytes", C.c_uint64)]


class SwapStats(C.Structure):
    _fields_ = [("bytes_d2h", C.c_uint64), ("bytes_h2d", C.c_uint64), ("chunks_d2h", C.c_uint32),
                ("chunks_h2d", C.c_uint32), ("ms", C.c_float), ("duplex", C.c_uint32)]


class StepTiming(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("complete_ms", "register_ms", "scan_ms", "select_ms",
                                           "finalize_ms", "total_ms")]


class StepStats(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("qstar", "mprime", "n_x", "n_b", "n_rows", "n_programs")] + \
               [("queue_counts", C.c_uint32 * 16)]


CALL_DESC = np.dtype([("call_id", "<u8"), ("program_id", "<u8"), ("arrival_step", "<u4"),
                      ("program_arrival_step", "<u4"), ("input_tokens", "<u4"), ("_pad", "<u4")])
CALL_STATE = np.dtype([("call_id", "<u8"), ("q", "<u4"), ("quanta", "<u4"), ("wait", "<u4"),
                       ("mtime", "<u4"), ("exec", "<u4"), ("totwait", "<u4"), ("inh", "<u4"),
                       ("input_tokens", "<u4"), ("arrival_step", "<u4"), ("flags", "<u4")])

_lib = None


def load_library(path=LIB_PATH):
    """Loads libautx.so; raises if it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    P = C.c_void_p
    u32, u64, i32 = C.c_uint32, C.c_uint64, C.c_int32
    sig = {
        "autx_create": ([C.POINTER(Config), C.POINTER(P)], i32),
        "autx_destroy": ([P], i32),
        "autx_last_error": ([P], C.c_char_p),
        "autx_version": ([], C.c_char_p),
        "autx_start_program": ([P, u64], i32),
        "autx_end_program": ([P, u64], i32),
        "autx_complete": ([P, P, u32], i32),
        "autx_register_call": ([P, P, u32], i32),
        "autx_register_call_dag": ([P, P, u32, P, P], i32),
        "autx_sched_step": ([P, u32, C.POINTER(StepOut)], i32),
        "autx_step_wait": ([P, C.POINTER(StepOut)], i32),
        "autx_step": ([P, u32, P, u32, P, u32, P, u32, C.POINTER(StepOut)], i32),
        "autx_kv_swap": ([P, C.POINTER(KvLayout), i32, C.POINTER(SwapStats)], i32),
        "autx_block_table": ([P, C.POINTER(P), C.POINTER(P)], i32),
        "autx_block_table_host": ([P, P, P, u32, C.POINTER(u32)], i32),
        "autx_route_record_bytes": ([P], u64),
        "autx_route_pack": ([P, P], i32),
        "autx_route_apply": ([P, P, P, u32, P], i32),
        "autx_route": ([P, P, u32, P], i32),
        "autx_comm_unique_id": ([P], i32),
        "autx_comm_init": ([P, i32, i32, i32, C.POINTER(P)], i32),
        "autx_comm_destroy": ([P], i32),
        "autx_dump_calls": ([P, P, u32, C.POINTER(u32)], i32),
        "autx_program_state": ([P, u64, C.POINTER(u32), C.POINTER(u64)], i32),
        "autx_last_step_timing": ([P, C.POINTER(StepTiming)], i32),
        "autx_step_stats": ([P, C.POINTER(StepStats)], i32),
        "autx_set_timing": ([P, i32], i32),
        "autx_num_active": ([P], u32),
        "autx_phase_times": ([P, P, u32], i32),
        "autx_kernel_launches": ([], u64),
        "autx_compaction_stats": ([P, C.POINTER(u64), C.POINTER(C.c_double)], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def exported_symbols():
    return [
        "autx_create", "autx_destroy", "autx_last_error", "autx_version", "autx_start_program",
        "autx_end_program", "autx_complete", "autx_register_call", "autx_register_call_dag", "autx_sched_step",
        "autx_step_wait", "autx_step", "autx_kv_swap", "autx_block_table", "autx_block_table_host", "autx_route_record_bytes",
        "autx_route_pack", "autx_route_apply", "autx_route", "autx_comm_unique_id", "autx_comm_init",
        "autx_comm_destroy", "autx_dump_calls", "autx_program_state",
        "autx_last_step_timing", "autx_step_stats", "autx_set_timing", "autx_num_active", "autx_phase_times", "autx_kernel_launches",
        "autx_compaction_stats"]


def kernel_launches():
    """Kernels launched by libautx.so so far in this process."""
    return int(load_library().autx_kernel_launches())


def comm_unique_id():
    """128-byte NCCL unique id (rank 0; broadcast it to the other ranks by any channel)."""
    buf = C.create_string_buffer(128)
    st = load_library().autx_comm_unique_id(buf)
    if st != 0:
        raise AutxError(st, "autx_comm_unique_id failed")
    return buf.raw


def comm_init(uid, rank, nranks, device):
    """The library's own NCCL communicator for autx_config.nccl_comm (collective over ranks)."""
    comm = C.c_void_p()
    st = load_library().autx_comm_init(C.create_string_buffer(bytes(uid), 128), rank, nranks, device,
                                       C.byref(comm))
    if st != 0:
        raise AutxError(st, "autx_comm_init failed")
    return comm.value


def comm_destroy(comm):
    if comm:
        load_library().autx_comm_destroy(C.c_void_p(comm))


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None and len(a) else C.c_void_p(0)


class Scheduler:
    """One engine's scheduler context (autx_ctx) on one GPU."""

    def __init__(self, policy="plas", K=1, q_hi=(), quanta=(None,), beta=(1, 0), max_batch=2,
                 kv_budget=None, block_tokens=16, max_calls=1 << 16, max_programs=1 << 16,
                 token_threshold=2048, order_mode=ORDER_SELECT, n_gpu_blocks=0,
                 max_blocks_per_call=0, host_pages=0, device=0, stream=None, rank=0, nranks=1,
                 route_policy="locality", nccl_comm=None, sched_every=1, overprovision=0):
        self.lib = load_library()
        cfg = Config()
        cfg.policy = POLICY[policy] if isinstance(policy, str) else int(policy)
        cfg.K = K
        for i, h in enumerate(q_hi):
            cfg.q_hi[i] = h
        for i, q in enumerate(quanta):
            cfg.quanta[i] = INF if q is None else q
        cfg.beta_num, cfg.beta_den = beta
        cfg.max_batch = max_batch
        cfg.kv_budget_blocks = INF if kv_budget is None else kv_budget
        cfg.block_tokens = block_tokens
        cfg.max_calls = max_calls
        cfg.max_programs = max_programs
        cfg.token_threshold = token_threshold
        cfg.order_mode = order_mode
        cfg.n_gpu_blocks = n_gpu_blocks
        cfg.max_blocks_per_call = max_blocks_per_call
        cfg.host_pages = host_pages
        cfg.device = device
        cfg.stream = stream
        cfg.rank, cfg.nranks = rank, nranks
        cfg.route_policy = ROUTE[route_policy] if isinstance(route_policy, str) else int(route_policy)
        cfg.nccl_comm = nccl_comm
        cfg.sched_every, cfg.overprovision = sched_every, overprovision   # R32
        self.cfg = cfg
        self.eq2 = cfg.policy == ATLAS_EQ2
        self.ctx = C.c_void_p()
        st = self.lib.autx_create(C.byref(cfg), C.byref(self.ctx))
        if st != 0:
            raise AutxError(st, "autx_create failed (see stderr)")
        self.out = StepOut()
        self.max_batch = max_batch
        self.list_cap = max_batch + overprovision
        self._views = None

    def _check(self, st):
        if st != 0:
            raise AutxError(st, self.lib.autx_last_error(self.ctx).decode())

    def close(self):
        if self.ctx:
            self.lib.autx_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- per-step calls ----------------------------------------------------------------
    def start_program(self, pid):
        self._check(self.lib.autx_start_program(self.ctx, int(pid)))

    def end_program(self, pid):
        self._check(self.lib.autx_end_program(self.ctx, int(pid)))

    def complete(self, call_ids):
        a = np.ascontiguousarray(call_ids, dtype=np.uint64)
        self._check(self.lib.autx_complete(self.ctx, _ptr(a), len(a)))

    def register(self, descs):
        """descs: structured array of CALL_DESC in canonical order."""
        a = np.ascontiguousarray(descs, dtype=CALL_DESC)
        self._check(self.lib.autx_register_call(self.ctx, _ptr(a), len(a)))

    def register_dag(self, descs, parent_offsets, parent_ids):
        """AUTX_ATLAS_EQ2 arrivals with their DAG parents (CSR: offsets[n+1] into parent ids)."""
        a = np.ascontiguousarray(descs, dtype=CALL_DESC)
        off = np.ascontiguousarray(parent_offsets, dtype=np.uint32)
        ids = np.ascontiguousarray(parent_ids, dtype=np.uint64)
        assert len(off) == len(a) + 1
        self._check(self.lib.autx_register_call_dag(self.ctx, _ptr(a), len(a), _ptr(off), _ptr(ids)))

    def sched_step(self, t, wait=True):
        self._check(self.lib.autx_sched_step(self.ctx, int(t), C.byref(self.out)))
        if wait:
            self._check(self.lib.autx_step_wait(self.ctx, C.byref(self.out)))
        return self.out

    def step(self, t, call_ids=None, ended_programs=(), descs=None):
        """One whole step in one ABI call (autx_step): completions, session ends, arrivals,
        sched_step and wait.  Returns the filled step record."""
        c = np.ascontiguousarray(call_ids if call_ids is not None else (), dtype=np.uint64)
        e = np.ascontiguousarray(ended_programs, dtype=np.uint64)
        a = np.ascontiguousarray(descs if descs is not None else np.zeros(0, CALL_DESC), dtype=CALL_DESC)
        self._check(self.lib.autx_step(self.ctx, int(t), _ptr(c), len(c), _ptr(e), len(e), _ptr(a), len(a),
                                       C.byref(self.out)))
        return self.out

    def step_wait(self):
        self._check(self.lib.autx_step_wait(self.ctx, C.byref(self.out)))
        return self.out

    def lists(self):
        """(batch, admit, preempt) call-id arrays of the last waited step (copies)."""
        o = self.out
        if self._views is None:
            # the pinned mirrors live as long as the context: wrap them once
            f = lambda p: np.ctypeslib.as_array(p, shape=(max(self.list_cap, 1),))
            self._views = (f(o.h_batch), f(o.h_admit), f(o.h_preempt))
        vb, va, vp = self._views
        return vb[:o.n_batch].copy(), va[:o.n_admit].copy(), vp[:o.n_preempt].copy()

    def compaction_stats(self):
        """(number of G8 compactions so far, host microseconds they took)."""
        n, us = C.c_uint64(), C.c_double()
        self._check(self.lib.autx_compaction_stats(self.ctx, C.byref(n), C.byref(us)))
        return int(n.value), float(us.value)

    def standby(self):
        """R32: the resident standby calls of the last waited step, in order (after the batch)."""
        self.lists()
        o = self.out
        return self._views[0][o.n_batch:o.n_batch + o.n_standby].copy()

    def kv_swap(self, k_ptrs, v_ptrs, chunk_bytes, host_ptr, host_bytes, mode=SWAP_STAGED_DMA):
        L = len(k_ptrs)
        kp = (C.c_void_p * L)(*k_ptrs)
        vp = (C.c_void_p * L)(*v_ptrs)
        lay = KvLayout(C.cast(kp, C.POINTER(C.c_void_p)), C.cast(vp, C.POINTER(C.c_void_p)), L,
                       chunk_bytes, C.c_void_p(host_ptr), host_bytes)
        st = SwapStats()
        self._check(self.lib.autx_kv_swap(self.ctx, C.byref(lay), mode, C.byref(st)))
        return st

    def block_table(self):
        o, b = C.c_void_p(), C.c_void_p()
        self._check(self.lib.autx_block_table(self.ctx, C.byref(o), C.byref(b)))
        return o.value, b.value

    def block_table_host(self, cap=1 << 22):
        """(offsets[n_batch+1], blocks) of the last batch as numpy arrays."""
        off = np.zeros(self.max_batch + 1, np.uint32)
        blk = np.zeros(cap, np.uint32)
        n = C.c_uint32()
        self._check(self.lib.autx_block_table_host(self.ctx, _ptr(off), _ptr(blk), cap, C.byref(n)))
        off = off[:n.value + 1]
        return off, blk[:off[-1]].copy()

    # ---- routing --------------------------------------------------------------------------
    def route_record_bytes(self):
        return int(self.lib.autx_route_record_bytes(self.ctx))

    def route_pack(self, d_record_ptr):
        self._check(self.lib.autx_route_pack(self.ctx, C.c_void_p(d_record_ptr)))

    def route_apply(self, d_records_ptr, descs):
        a = np.ascontiguousarray(descs, dtype=CALL_DESC)
        out = np.zeros(len(a), np.int32)
        self._check(self.lib.autx_route_apply(self.ctx, C.c_void_p(d_records_ptr), _ptr(a), len(a),
                                              _ptr(out)))
        return out

    def route(self, descs):
        """One routing epoch as one collective (autx_route): record, NCCL all-gather, apply, Alg. 2."""
        a = np.ascontiguousarray(descs, dtype=CALL_DESC)
        out = np.zeros(len(a), np.int32)
        self._check(self.lib.autx_route(self.ctx, _ptr(a), len(a), _ptr(out)))
        return out

    # ---- introspection ----------------------------------------------------------------------
    def dump_calls(self):
        n = C.c_uint32()
        self._check(self.lib.autx_dump_calls(self.ctx, None, 0, C.byref(n)))
        a = np.zeros(n.value, CALL_STATE)
        self._check(self.lib.autx_dump_calls(self.ctx, _ptr(a), n.value, C.byref(n)))
        return a

    def program_state(self, pid):
        s, w = C.c_uint32(), C.c_uint64()
        self._check(self.lib.autx_program_state(self.ctx, int(pid), C.byref(s), C.byref(w)))
        return s.value, w.value

    def step_stats(self):
        """Selection shape of the last step: q*, m', region A / B sizes, rows, programs, queues."""
        st = StepStats()
        self._check(self.lib.autx_step_stats(self.ctx, C.byref(st)))
        d = {n: int(getattr(st, n)) for n, _ in StepStats._fields_[:6]}
        d["queue_counts"] = [int(x) for x in st.queue_counts]
        return d

    def set_timing(self, on=True, stamps=False):
        """on: CUDA events around the step's kernels; stamps: %globaltimer phase stamps inside
        the step kernel instead (read with phase_times())."""
        self._check(self.lib.autx_set_timing(self.ctx, (1 if on else 0) | (2 if stamps else 0)))

    def last_step_timing(self):
        t = StepTiming()
        self._check(self.lib.autx_last_step_timing(self.ctx, C.byref(t)))
        return t

    def phase_times(self):
        a = np.zeros(96, np.uint64)
        self._check(self.lib.autx_phase_times(self.ctx, _ptr(a), 96))
        return a

    def num_active(self):
        return int(self.lib.autx_num_active(self.ctx))
