"""Thin ctypes binding of libadaptis.so (include/adaptis.h).

Argument marshalling only: every step of the hot path (decode, stage sums,
simulation, argmin) runs in the library's CUDA kernels. PyTorch is used for
device memory, streams and torch.distributed (the allreduce hook), nothing
else. There is no CPU fallback: if libadaptis.so is missing or has no GPU to
run on, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import threading
from typing import Optional

import numpy as np

from . import workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libadaptis.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "adaptis.h")
MAX_P, MAX_V, MAX_S, MAX_GROUPS = 32, 4, 64, 4
INT64_MAX = (1 << 63) - 1
UINT64_MAX = (1 << 64) - 1

OK, EINVAL, EINFEASIBLE, EOVERFLOW, ECUDA, ECOLL = range(6)


class AdaptisError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s (status %d)" % (msg, status))
        self.status = status


class _Layers(C.Structure):
    _fields_ = [("L", C.c_int32)] + [(n, C.POINTER(C.c_int64)) for n in (
        "t_f", "t_b", "t_w", "act_bytes", "stash_bytes", "weight_bytes", "grad_bytes", "comm_ticks")]


class _Problem(C.Structure):
    _fields_ = [("layers", _Layers), ("p", C.c_int32), ("m", C.c_int32),
                ("mem_cap_bytes", C.c_int64), ("tick_seconds", C.c_double),
                ("tokens_per_microbatch", C.c_int64), ("cost_type", C.c_int32),
                ("costs_f32", C.POINTER(C.c_float))]


class _Group(C.Structure):
    _fields_ = [("v", C.c_int32), ("part_mode", C.c_int32), ("radius", C.c_int32),
                ("seed_cuts", C.POINTER(C.c_int16)), ("combo_mask", C.c_uint32)]


class _Space(C.Structure):
    _fields_ = [("n_groups", C.c_int32), ("group", _Group * MAX_GROUPS)]


class _Plan(C.Structure):
    _fields_ = [("v", C.c_int32), ("placement", C.c_int32), ("policy", C.c_int32),
                ("S", C.c_int32), ("cuts", C.c_int16 * (MAX_S + 1))]


class _ResultsSoa(C.Structure):
    _fields_ = [("makespan", C.c_void_p), ("peak_mem_bytes", C.c_void_p),
                ("bubble_ratio", C.c_void_p), ("status", C.c_void_p), ("makespan_f32", C.c_void_p)]


class _Result(C.Structure):
    _fields_ = [("makespan", C.c_int64), ("peak_mem_bytes", C.c_int64),
                ("bubble_ratio", C.c_float), ("throughput", C.c_double), ("status", C.c_uint8),
                ("makespan_f32", C.c_float)]


ACCT = ("comm_d", "exposed_d", "overlap_d", "bubble_d")  # R29, Alg. 1 Step 3 accounting


class _Best(C.Structure):
    _fields_ = [("index", C.c_uint64), ("plan", _Plan), ("result", _Result), ("p", C.c_int32),
                ("T_d", C.c_int64 * MAX_P), ("busy_d", C.c_int64 * MAX_P),
                ("M_d", C.c_int64 * MAX_P)] + [(k, C.c_int64 * MAX_P) for k in ACCT] + [
                ("n_candidates", C.c_uint64),
                ("n_evaluated", C.c_uint64), ("n_invalid", C.c_uint64), ("n_tasks", C.c_uint64),
                ("n_pruned", C.c_uint64), ("kernel_ms", C.c_float)]


class _GenOptions(C.Structure):
    _fields_ = [("vs_mask", C.c_uint32), ("radius", C.c_int32), ("max_rounds", C.c_int32),
                ("mode", C.c_int32)]


GEN_MAX_STEPS = 128
GEN_PHASES = {0: "seed", 1: "partition", 2: "placement", 3: "schedule"}


class _GenResult(C.Structure):
    _fields_ = [("plan", _Plan), ("result", _Result), ("p", C.c_int32),
                ("T_d", C.c_int64 * MAX_P), ("busy_d", C.c_int64 * MAX_P),
                ("M_d", C.c_int64 * MAX_P)] + [(k, C.c_int64 * MAX_P) for k in ACCT] + [
                ("n_seeds", C.c_int32), ("rounds", C.c_int32),
                ("n_evaluated", C.c_uint64), ("n_steps", C.c_int32),
                ("step_phase", C.c_int32 * GEN_MAX_STEPS), ("step_makespan", C.c_int64 * GEN_MAX_STEPS),
                ("kernel_ms", C.c_float)]


class _MemPoint(C.Structure):
    _fields_ = [("time", C.c_int64), ("bytes", C.c_int64)]


class _LaunchInfo(C.Structure):
    _fields_ = [("group", C.c_int32), ("combo", C.c_int32), ("v", C.c_int32),
                ("placement", C.c_int32), ("policy", C.c_int32), ("fallback", C.c_int32),
                ("candidates", C.c_uint64), ("tasks", C.c_uint64), ("ms", C.c_float),
                ("kernel", C.c_int32)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)

_lock = threading.Lock()
_lib = None


def exported_symbols():
    """Entry points declared in include/adaptis.h."""
    src = open(HEADER).read()
    return sorted(set(re.findall(r"ADAPTIS_API\s+[\w\s\*]*?\b(adaptis_[a-z_]+)\s*\(", src)))


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError("libadaptis.so not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = C.CDLL(LIB_PATH)
            st = C.c_int
            L.adaptis_status_str.restype = C.c_char_p
            L.adaptis_last_error.restype = C.c_char_p
            L.adaptis_last_error.argtypes = [C.c_void_p]
            L.adaptis_ctx_create.restype = st
            L.adaptis_ctx_create.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
            L.adaptis_ctx_destroy.argtypes = [C.c_void_p]
            L.adaptis_ctx_set_prune.restype = st
            L.adaptis_ctx_set_prune.argtypes = [C.c_void_p, C.c_int]
            L.adaptis_ctx_set_allreduce.restype = st
            L.adaptis_ctx_set_allreduce.argtypes = [C.c_void_p, ALLREDUCE_FN, C.c_void_p]
            L.adaptis_ctx_stream.restype = C.c_void_p
            L.adaptis_ctx_stream.argtypes = [C.c_void_p]
            L.adaptis_ctx_launch_count.restype = C.c_uint64
            L.adaptis_ctx_launch_count.argtypes = [C.c_void_p]
            L.adaptis_ctx_fallback_count.restype = C.c_uint64
            L.adaptis_ctx_fallback_count.argtypes = [C.c_void_p]
            L.adaptis_ctx_counters.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
            L.adaptis_ctx_launch_info.restype = C.c_int
            L.adaptis_ctx_launch_info.argtypes = [C.c_void_p, C.POINTER(_LaunchInfo), C.c_int]
            L.adaptis_static_order.restype = st
            L.adaptis_static_order.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                               C.POINTER(C.c_uint32), C.c_uint64, C.POINTER(C.c_uint64),
                                               C.POINTER(C.c_int32)]
            L.adaptis_space_size.restype = st
            L.adaptis_space_size.argtypes = [C.POINTER(_Problem), C.POINTER(_Space), C.POINTER(C.c_uint64)]
            L.adaptis_decode.restype = st
            L.adaptis_decode.argtypes = [C.POINTER(_Problem), C.POINTER(_Space), C.c_uint64, C.POINTER(_Plan)]
            L.adaptis_prepare.restype = st
            L.adaptis_prepare.argtypes = [C.c_void_p, C.POINTER(_Problem), C.POINTER(_Space),
                                          C.POINTER(C.c_void_p)]
            L.adaptis_prepared_free.argtypes = [C.c_void_p]
            L.adaptis_eval_batch.restype = st
            L.adaptis_eval_batch.argtypes = [C.c_void_p, C.POINTER(_Problem), C.POINTER(_Space),
                                             C.c_uint64, C.c_uint64, C.POINTER(_ResultsSoa), C.c_int]
            L.adaptis_eval_prepared.restype = st
            L.adaptis_eval_prepared.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                                C.POINTER(_ResultsSoa), C.c_int]
            L.adaptis_shard_indices.restype = st
            L.adaptis_shard_indices.argtypes = [C.POINTER(_Problem), C.POINTER(_Space), C.c_int, C.c_int,
                                                C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(C.c_uint64)]
            L.adaptis_search.restype = st
            L.adaptis_search.argtypes = [C.c_void_p, C.POINTER(_Problem), C.POINTER(_Space), C.POINTER(_Best)]
            L.adaptis_search_prepared.restype = st
            L.adaptis_search_prepared.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Best)]
            L.adaptis_eval_indices.restype = st
            L.adaptis_eval_indices.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64,
                                               C.POINTER(_ResultsSoa)]
            L.adaptis_eval_lists.restype = st
            L.adaptis_eval_lists.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Plan), C.c_void_p,
                                             C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(_ResultsSoa),
                                             C.POINTER(C.c_int64)]
            L.adaptis_eval_lists_contended.restype = st
            L.adaptis_eval_lists_contended.argtypes = L.adaptis_eval_lists.argtypes
            L.adaptis_repair_oom.restype = st
            L.adaptis_repair_oom.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Plan), C.c_void_p,
                                             C.POINTER(C.c_uint64), C.c_int32, C.c_void_p,
                                             C.POINTER(_Result), C.POINTER(C.c_int32)]
            L.adaptis_tune_overlap.restype = st
            L.adaptis_tune_overlap.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Plan), C.c_void_p,
                                               C.POINTER(C.c_uint64), C.c_int32, C.c_void_p,
                                               C.POINTER(_Result), C.POINTER(C.c_int32),
                                               C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
            L.adaptis_eval_contended.restype = st
            L.adaptis_eval_contended.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                                 C.POINTER(_ResultsSoa)]
            L.adaptis_search_contended.restype = st
            L.adaptis_search_contended.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Best)]
            L.adaptis_realize_lists.restype = st
            L.adaptis_realize_lists.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Plan), C.c_void_p,
                                                C.c_uint64, C.POINTER(C.c_uint64)]
            L.adaptis_memory_timeline.restype = st
            L.adaptis_memory_timeline.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Plan), C.c_void_p,
                                                  C.POINTER(C.c_uint64), C.POINTER(_MemPoint), C.c_uint64,
                                                  C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]
            L.adaptis_lower.restype = st
            L.adaptis_lower.argtypes = [C.c_int32, C.POINTER(_Plan), C.c_void_p, C.POINTER(C.c_uint64),
                                        C.c_int32, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
            L.adaptis_lower_error.restype = C.c_char_p
            L.adaptis_eval_plans.restype = st
            L.adaptis_eval_plans.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Plan), C.c_uint64,
                                             C.POINTER(_ResultsSoa), C.POINTER(C.c_int64)]
            L.adaptis_generate.restype = st
            L.adaptis_generate.argtypes = [C.c_void_p, C.POINTER(_Problem), C.POINTER(_GenOptions),
                                           C.POINTER(_GenResult)]
            _lib = L
    return _lib


def _err(ctx_ptr=None) -> str:
    return (lib().adaptis_last_error(ctx_ptr) or b"").decode()


class _Marshal:
    """C views of a workloads.Problem / Space; keeps the numpy buffers alive."""

    def __init__(self, pr: W.Problem, sp: Optional[W.Space] = None):
        self.keep = []
        ptrs = {}
        for src, dst in (("t_f", "t_f"), ("t_b", "t_b"), ("t_w", "t_w"), ("act", "act_bytes"),
                         ("stash", "stash_bytes"), ("weight", "weight_bytes"),
                         ("grad", "grad_bytes"), ("comm", "comm_ticks")):
            a = np.ascontiguousarray(np.asarray(getattr(pr, src), dtype=np.int64))
            self.keep.append(a)
            ptrs[dst] = a.ctypes.data_as(C.POINTER(C.c_int64))
        cf = None
        if getattr(pr, "costs_f32", None) is not None:
            a = np.ascontiguousarray(np.asarray(pr.costs_f32, dtype=np.float32))
            self.keep.append(a)
            cf = a.ctypes.data_as(C.POINTER(C.c_float))
        self.problem = _Problem(layers=_Layers(L=len(pr.t_f), **ptrs), p=pr.p, m=pr.m,
                                mem_cap_bytes=int(pr.cap), tick_seconds=float(pr.tick_seconds),
                                tokens_per_microbatch=int(pr.tokens_per_microbatch),
                                cost_type=int(getattr(pr, "cost_type", 0)), costs_f32=cf)
        self.space = None
        if sp is not None:
            s = _Space(n_groups=len(sp.groups))
            for i, g in enumerate(sp.groups):
                seed = None
                if g.seed_cuts is not None:
                    arr = (C.c_int16 * len(g.seed_cuts))(*g.seed_cuts)
                    self.keep.append(arr)
                    seed = C.cast(arr, C.POINTER(C.c_int16))
                s.group[i] = _Group(v=g.v, part_mode=g.part_mode, radius=g.radius,
                                    seed_cuts=seed, combo_mask=g.combo_mask)
            self.space = s


def _check(status, ctx_ptr=None):
    if status != OK:
        raise AdaptisError(status, _err(ctx_ptr))


def plan_dict(pl: _Plan) -> dict:
    return {"v": pl.v, "placement": pl.placement, "policy": pl.policy, "S": pl.S,
            "cuts": [int(pl.cuts[i]) for i in range(pl.S + 1)]}


def make_plans(plans) -> "C.Array":
    """dicts {v, placement, policy, cuts (S+1 values or S-1 interior cuts)} -> adaptis_plan[]"""
    arr = (_Plan * max(1, len(plans)))()
    for i, d in enumerate(plans):
        S = int(d.get("S", 0)) or (len(d["cuts"]) - 1)
        cuts = list(d["cuts"])
        if len(cuts) == S - 1:
            cuts = [0] + cuts + [0]  # cuts[0] and cuts[S] are implied (0 and L)
        arr[i].v, arr[i].placement, arr[i].policy, arr[i].S = d["v"], d["placement"], d["policy"], S
        for k, c in enumerate(cuts[:S + 1]):
            arr[i].cuts[k] = int(c)
    return arr


LOWER_REPAIR, LOWER_HOIST = 1, 2


def lower(p: int, plan: dict, lists, repair: bool = True, hoist: bool = True) -> dict:
    """adaptis_lower (host only, R33): per-device Table-5 instruction programs of
    an explicit schedule, as lists of (op, stage, mb, peer)."""
    arr = make_plans([plan])
    tasks, offs = Prepared._task_arrays([lists], p)
    total = int(offs[p])
    cap = 4 * max(total, 1)
    out = np.zeros(cap, dtype=[("op", "<i4"), ("stage", "<i4"), ("mb", "<i4"), ("peer", "<i4")])
    ooff = np.zeros(p + 1, np.uint64)
    nr, nh = C.c_int32(), C.c_int32()
    flags = (LOWER_REPAIR if repair else 0) | (LOWER_HOIST if hoist else 0)
    st = lib().adaptis_lower(p, arr, tasks.ctypes.data, offs.ctypes.data_as(C.POINTER(C.c_uint64)), flags,
                             out.ctypes.data, cap, ooff.ctypes.data_as(C.POINTER(C.c_uint64)),
                             C.byref(nr), C.byref(nh))
    if st != OK:
        raise AdaptisError(st, (lib().adaptis_lower_error() or b"").decode())
    prog = [[tuple(int(x) for x in out[i]) for i in range(int(ooff[d]), int(ooff[d + 1]))] for d in range(p)]
    return {"programs": prog, "repairs": int(nr.value), "hoists": int(nh.value)}


def static_order(policy: int, placement: int, p: int, v: int, m: int):
    """The static-order kernel's task order of a GPIPE / ONEF1B / ZB segment
    (host-only entry point): a list of (stage, kind, in_slot, out_slot,
    device) with slot None for no item, and the number of slots."""
    n = C.c_uint64()
    ns = C.c_int32()
    cap = 2 * p * v * m  # 2 S m F/B entries
    buf = (C.c_uint32 * max(cap, 1))()
    _check(lib().adaptis_static_order(policy, placement, p, v, m, buf, cap, C.byref(n), C.byref(ns)))
    out = []
    for i in range(int(n.value)):
        e = int(buf[i])
        ins, outs = (e >> 8) & 255, (e >> 16) & 255
        out.append((e & 63, (e >> 6) & 1, None if ins == 255 else ins, None if outs == 255 else outs, (e >> 24) & 15))
    return out, int(ns.value)


def space_size(pr: W.Problem, sp: W.Space) -> int:
    """|space| (host-only entry point; no GPU needed)."""
    m = _Marshal(pr, sp)
    n = C.c_uint64()
    _check(lib().adaptis_space_size(C.byref(m.problem), C.byref(m.space), C.byref(n)))
    return int(n.value)


def decode(pr: W.Problem, sp: W.Space, index: int) -> dict:
    """Candidate index -> plan, canonical order R19 (host-only entry point)."""
    m = _Marshal(pr, sp)
    pl = _Plan()
    _check(lib().adaptis_decode(C.byref(m.problem), C.byref(m.space), index, C.byref(pl)))
    return plan_dict(pl)


def shard_indices(pr: W.Problem, sp: W.Space, rank: int, world: int) -> np.ndarray:
    """Global indices rank `rank` evaluates in a `world`-way sharded search (host-only)."""
    m = _Marshal(pr, sp)
    n = C.c_uint64()
    _check(lib().adaptis_shard_indices(C.byref(m.problem), C.byref(m.space), rank, world, None, 0,
                                       C.byref(n)))
    out = np.zeros(n.value, np.uint64)
    _check(lib().adaptis_shard_indices(C.byref(m.problem), C.byref(m.space), rank, world,
                                       out.ctypes.data_as(C.POINTER(C.c_uint64)), n.value, C.byref(n)))
    return out


def pack_key(makespan: int, index: int, n_candidates: int) -> int:
    """The packed argmin key of the search (makespan << bits | index)."""
    bits = max(1, (n_candidates - 1).bit_length())
    return (makespan << bits) | index


class Context:
    """One adaptis_ctx bound to a CUDA device (and a rank of a sharded search)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, group=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("adaptis needs a CUDA device (no CPU fallback)")
        torch.cuda.init()
        self.device = device
        self.ptr = C.c_void_p()
        _check(lib().adaptis_ctx_create(device, rank, world, C.byref(self.ptr)))
        self._cb = None
        self._group = group
        if world > 1:
            self._install_allreduce(group)

    def _install_allreduce(self, group):
        import torch
        import torch.distributed as dist
        dev = self.device

        def _allreduce(dev_key, stream, _user):
            try:
                # zero-copy view of the 8-byte key in device memory
                buf = _device_int64_view(dev_key, dev)
                t = torch.empty(1, dtype=torch.int64, device="cuda:%d" % dev)
                ext = torch.cuda.ExternalStream(stream, device=dev)
                with torch.cuda.stream(ext):
                    t.copy_(buf)
                    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
                    buf.copy_(t)
                ext.synchronize()
                return 0
            except Exception as e:  # noqa: BLE001 - reported as ADAPTIS_ECOLL
                import sys
                print("adaptis allreduce failed:", repr(e), file=sys.stderr)
                return 1

        self._cb = ALLREDUCE_FN(_allreduce)
        _check(lib().adaptis_ctx_set_allreduce(self.ptr, self._cb, None), self.ptr)

    def set_prune(self, enable: bool = True):
        """Exact lower-bound pruning for search (winner unchanged; see adaptis.h)."""
        _check(lib().adaptis_ctx_set_prune(self.ptr, int(bool(enable))), self.ptr)

    @property
    def stream(self) -> int:
        return lib().adaptis_ctx_stream(self.ptr)

    @property
    def launch_count(self) -> int:
        return int(lib().adaptis_ctx_launch_count(self.ptr))

    @property
    def counters(self) -> dict:
        a = (C.c_uint64 * 3)()
        lib().adaptis_ctx_counters(self.ptr, a)
        return {"tasks": int(a[0]), "rounds": int(a[1]), "live_lane_rounds": int(a[2])}

    def launch_info(self) -> list:
        """Per-segment launches of the last evaluation (device ms via CUDA events)."""
        arr = (_LaunchInfo * 64)()
        n = lib().adaptis_ctx_launch_info(self.ptr, arr, 64)
        return [{k: getattr(arr[i], k) for k, _ in _LaunchInfo._fields_} for i in range(min(n, 64))]

    @property
    def fallback_count(self) -> int:
        return int(lib().adaptis_ctx_fallback_count(self.ptr))

    def close(self):
        if self.ptr:
            lib().adaptis_ctx_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # ------------------------------------------------------------------
    def prepare(self, pr: W.Problem, sp: W.Space) -> "Prepared":
        return Prepared(self, pr, sp)

    def eval_batch(self, pr: W.Problem, sp: W.Space, first: int, count: int) -> dict:
        """Per-candidate results for [first, first+count), host buffers (e2e path)."""
        m = _Marshal(pr, sp)
        out = _host_results(count)
        soa = _soa_from_numpy(out)
        _check(lib().adaptis_eval_batch(self.ptr, C.byref(m.problem), C.byref(m.space), first, count,
                                        C.byref(soa), 0), self.ptr)
        return out

    def search(self, pr: W.Problem, sp: W.Space) -> dict:
        """adaptis_search with host inputs (validate + upload + evaluate + reduce)."""
        m = _Marshal(pr, sp)
        b = _Best()
        st = lib().adaptis_search(self.ptr, C.byref(m.problem), C.byref(m.space), C.byref(b))
        return _best_dict(b, st, self.ptr)

    def generate(self, pr: W.Problem, vs_mask: int = 0, radius: int = 0, max_rounds: int = 0,
                 mode: str = "bottleneck") -> dict:
        """adaptis_generate: the Pipeline Generator (R28' / R28) on this GPU."""
        m = _Marshal(pr)
        o = _GenOptions(vs_mask=vs_mask, radius=radius, max_rounds=max_rounds,
                        mode={"bottleneck": 0, "round-robin": 1}[mode])
        r = _GenResult()
        st = lib().adaptis_generate(self.ptr, C.byref(m.problem), C.byref(o), C.byref(r))
        if st not in (OK, EINFEASIBLE):
            raise AdaptisError(st, _err(self.ptr))
        p = r.p
        n = r.n_steps
        return {"status": st, "plan": plan_dict(r.plan), "makespan": int(r.result.makespan),
                "peak_mem": int(r.result.peak_mem_bytes), "bubble": float(r.result.bubble_ratio),
                "throughput": float(r.result.throughput), "cand_status": int(r.result.status),
                "T_d": list(r.T_d[:p]), "busy_d": list(r.busy_d[:p]), "M_d": list(r.M_d[:p]),
                **{k: list(getattr(r, k)[:p]) for k in ACCT},
                "n_seeds": int(r.n_seeds), "rounds": int(r.rounds), "n_evaluated": int(r.n_evaluated),
                "steps": [(GEN_PHASES[int(r.step_phase[i])], int(r.step_makespan[i])) for i in range(n)],
                "kernel_ms": float(r.kernel_ms)}


class Prepared:
    """Problem tables resident in HBM (adaptis_prepare) for repeated evaluation."""

    def __init__(self, ctx: Context, pr: W.Problem, sp: W.Space):
        self.ctx = ctx
        self.m = _Marshal(pr, sp)
        self.ptr = C.c_void_p()
        _check(lib().adaptis_prepare(ctx.ptr, C.byref(self.m.problem), C.byref(self.m.space),
                                     C.byref(self.ptr)), ctx.ptr)
        self.N = space_size(pr, sp)

    def close(self):
        if self.ptr:
            lib().adaptis_prepared_free(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def search(self) -> dict:
        b = _Best()
        st = lib().adaptis_search_prepared(self.ctx.ptr, self.ptr, C.byref(b))
        return _best_dict(b, st, self.ctx.ptr)

    def eval_indices(self, indices) -> dict:
        """adaptis_eval_indices: results for arbitrary global indices (device decode)."""
        idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
        out = _host_results(len(idx))
        soa = _soa_from_numpy(out)
        _check(lib().adaptis_eval_indices(self.ctx.ptr, self.ptr, idx.ctypes.data_as(C.POINTER(C.c_uint64)),
                                          len(idx), C.byref(soa)), self.ctx.ptr)
        return out

    def eval_plans(self, plans, report: bool = False) -> dict:
        """adaptis_eval_plans: results (and optionally T_d/busy_d/M_d) of explicit plans."""
        n = len(plans)
        arr = make_plans(plans)
        out = _host_results(n)
        soa = _soa_from_numpy(out)
        rep = np.zeros((max(n, 1), REPORT_ROWS, self.m.problem.p), np.int64) if report else None
        _check(lib().adaptis_eval_plans(self.ctx.ptr, self.ptr, arr, n, C.byref(soa),
                                        rep.ctypes.data_as(C.POINTER(C.c_int64)) if report else None),
               self.ctx.ptr)
        if report:
            _unpack_report(out, rep, n)
        return out

    def eval_lists_contended(self, plans, lists, report: bool = False) -> dict:
        """adaptis_eval_lists_contended: eval_lists with FIFO send / receive
        engines per device (R34)."""
        return self.eval_lists(plans, lists, report, _contended=True)

    def eval_lists(self, plans, lists, report: bool = False, _contended: bool = False) -> dict:
        """adaptis_eval_lists: plans (policy LIST = 4 / LIST_FUSED = 5) with explicit
        per-device orders lists[i][d] = [(kind, stage, mb), ...] (R30)."""
        n = len(plans)
        p = self.m.problem.p
        arr = make_plans(plans)
        flat = [t for per_plan in lists for dev in per_plan for t in dev]
        tasks = np.zeros(max(1, len(flat)), dtype=[("kind", "<i2"), ("stage", "<i2"), ("mb", "<i4")])
        for q, (k, s_, j) in enumerate(flat):
            tasks[q] = (k, s_, j)
        offs = np.zeros(max(1, n * (p + 1)), np.uint64)
        pos = 0
        for i, per_plan in enumerate(lists):
            for d in range(p):
                offs[i * (p + 1) + d] = pos
                pos += len(per_plan[d])
            offs[i * (p + 1) + p] = pos
        out = _host_results(n)
        soa = _soa_from_numpy(out)
        rep = np.zeros((max(n, 1), REPORT_ROWS, p), np.int64) if report else None
        fn = lib().adaptis_eval_lists_contended if _contended else lib().adaptis_eval_lists
        _check(fn(self.ctx.ptr, self.ptr, arr, tasks.ctypes.data,
                                        offs.ctypes.data_as(C.POINTER(C.c_uint64)), n, C.byref(soa),
                                        rep.ctypes.data_as(C.POINTER(C.c_int64)) if report else None),
               self.ctx.ptr)
        if report:
            _unpack_report(out, rep, n)
        return out

    @staticmethod
    def _task_arrays(lists_per_plan, p):
        flat = [t for per_plan in lists_per_plan for dev in per_plan for t in dev]
        tasks = np.zeros(max(1, len(flat)), dtype=[("kind", "<i2"), ("stage", "<i2"), ("mb", "<i4")])
        for q, (k, s_, j) in enumerate(flat):
            tasks[q] = (k, s_, j)
        offs = np.zeros(max(1, len(lists_per_plan) * (p + 1)), np.uint64)
        pos = 0
        for i, per_plan in enumerate(lists_per_plan):
            for d in range(p):
                offs[i * (p + 1) + d] = pos
                pos += len(per_plan[d])
            offs[i * (p + 1) + p] = pos
        return tasks, offs

    def repair_oom(self, plan, lists, max_moves: int = 0) -> dict:
        """adaptis_repair_oom (R31): the repaired per-device lists and their result."""
        p = self.m.problem.p
        arr = make_plans([plan])
        tasks, offs = self._task_arrays([lists], p)
        out_tasks = np.zeros_like(tasks)
        res = _Result()
        nm = C.c_int32()
        _check(lib().adaptis_repair_oom(self.ctx.ptr, self.ptr, arr, tasks.ctypes.data,
                                        offs.ctypes.data_as(C.POINTER(C.c_uint64)), max_moves,
                                        out_tasks.ctypes.data, C.byref(res), C.byref(nm)), self.ctx.ptr)
        rep = [[(int(t["kind"]), int(t["stage"]), int(t["mb"])) for t in out_tasks[int(offs[d]):int(offs[d + 1])]]
               for d in range(p)]
        return {"lists": rep, "moves": int(nm.value), "status": int(res.status),
                "makespan": int(res.makespan), "peak_mem": int(res.peak_mem_bytes)}

    def eval_contended(self, first: int, count: int) -> dict:
        """adaptis_eval_contended (R36): results of [first, first + count) when each
        candidate's realised order runs under send/receive-engine contention."""
        out = _host_results(count)
        soa = _soa_from_numpy(out)
        _check(lib().adaptis_eval_contended(self.ctx.ptr, self.ptr, first, count, C.byref(soa)), self.ctx.ptr)
        return out

    def search_contended(self) -> dict:
        """adaptis_search_contended (R36): the argmin of the contended makespans."""
        b = _Best()
        st = lib().adaptis_search_contended(self.ctx.ptr, self.ptr, C.byref(b))
        if st not in (OK, EINFEASIBLE):
            raise AdaptisError(st, _err(self.ctx.ptr))
        return _best_dict(b, st, self.ctx.ptr)

    def realize_lists(self, plan) -> list:
        """adaptis_realize_lists: the plan's realised per-device orders (R30 lists
        of (kind, stage, mb); fused policies without W)."""
        p, m = self.m.problem.p, self.m.problem.m
        arr = make_plans([plan])
        cap = p * 3 * m * plan["v"]
        tasks = np.zeros(cap, dtype=[("kind", "<i2"), ("stage", "<i2"), ("mb", "<i4")])
        offs = (C.c_uint64 * (p + 1))()
        _check(lib().adaptis_realize_lists(self.ctx.ptr, self.ptr, arr, tasks.ctypes.data, cap, offs),
               self.ctx.ptr)
        return [[tuple(int(x) for x in tasks[i]) for i in range(offs[d], offs[d + 1])] for d in range(p)]

    def memory_timeline(self, plan, lists=None) -> dict:
        """adaptis_memory_timeline (R35): per device the breakpoints (time, bytes)
        of static + dynamic memory and the first time above the cap (-1: never)."""
        p, m = self.m.problem.p, self.m.problem.m
        arr = make_plans([plan])
        cap = p * (1 + 3 * m * plan["v"])
        out = (_MemPoint * cap)()
        offs = (C.c_uint64 * (p + 1))()
        first = (C.c_int64 * p)()
        if lists is not None:
            tasks, toffs = self._task_arrays([lists], p)
            st = lib().adaptis_memory_timeline(self.ctx.ptr, self.ptr, arr, tasks.ctypes.data,
                                               toffs.ctypes.data_as(C.POINTER(C.c_uint64)), out, cap,
                                               offs, first)
        else:
            st = lib().adaptis_memory_timeline(self.ctx.ptr, self.ptr, arr, None, None, out, cap, offs, first)
        _check(st, self.ctx.ptr)
        pts = [[(int(out[i].time), int(out[i].bytes)) for i in range(offs[d], offs[d + 1])] for d in range(p)]
        return {"points": pts, "first_violation": [int(x) for x in first]}

    def tune_overlap(self, plan, lists, max_swaps: int = 0) -> dict:
        """adaptis_tune_overlap (R32): the reordered lists and their result."""
        p = self.m.problem.p
        arr = make_plans([plan])
        tasks, offs = self._task_arrays([lists], p)
        out_tasks = np.zeros_like(tasks)
        res = _Result()
        ns = C.c_int32()
        ob, oa = C.c_int64(), C.c_int64()
        _check(lib().adaptis_tune_overlap(self.ctx.ptr, self.ptr, arr, tasks.ctypes.data,
                                          offs.ctypes.data_as(C.POINTER(C.c_uint64)), max_swaps,
                                          out_tasks.ctypes.data, C.byref(res), C.byref(ns),
                                          C.byref(ob), C.byref(oa)), self.ctx.ptr)
        out = [[(int(t["kind"]), int(t["stage"]), int(t["mb"])) for t in out_tasks[int(offs[d]):int(offs[d + 1])]]
               for d in range(p)]
        return {"lists": out, "swaps": int(ns.value), "status": int(res.status),
                "makespan": int(res.makespan), "overlap_before": int(ob.value), "overlap_after": int(oa.value)}

    def eval(self, first: int, count: int, device_out: bool = False):
        """Results for [first, first+count): numpy (host) or torch CUDA tensors."""
        if device_out:
            import torch
            dev = "cuda:%d" % self.ctx.device
            out = {"makespan": torch.empty(count, dtype=torch.int64, device=dev),
                   "peak_mem": torch.empty(count, dtype=torch.int64, device=dev),
                   "bubble": torch.empty(count, dtype=torch.float32, device=dev),
                   "status": torch.empty(count, dtype=torch.uint8, device=dev),
                   "makespan_f32": torch.empty(count, dtype=torch.float32, device=dev)}
            soa = _ResultsSoa(out["makespan"].data_ptr(), out["peak_mem"].data_ptr(),
                              out["bubble"].data_ptr(), out["status"].data_ptr(),
                              out["makespan_f32"].data_ptr())
            torch.cuda.current_stream(self.ctx.device).synchronize()
            _check(lib().adaptis_eval_prepared(self.ctx.ptr, self.ptr, first, count, C.byref(soa), 1),
                   self.ctx.ptr)
            return out
        out = _host_results(count)
        soa = _soa_from_numpy(out)
        _check(lib().adaptis_eval_prepared(self.ctx.ptr, self.ptr, first, count, C.byref(soa), 0),
               self.ctx.ptr)
        return out


REPORT_ROWS = 7  # adaptis.h per-plan report rows
REPORT_KEYS = ("T_d", "busy_d", "M_d", "comm_d", "exposed_d", "overlap_d", "bubble_d")


def _unpack_report(out, rep, n):
    for r, k in enumerate(REPORT_KEYS):
        out[k] = rep[:n, r]


def _host_results(count):
    return {"makespan": np.zeros(count, np.int64), "peak_mem": np.zeros(count, np.int64),
            "bubble": np.zeros(count, np.float32), "status": np.zeros(count, np.uint8),
            "makespan_f32": np.zeros(count, np.float32)}


def _soa_from_numpy(out):
    return _ResultsSoa(out["makespan"].ctypes.data, out["peak_mem"].ctypes.data,
                       out["bubble"].ctypes.data, out["status"].ctypes.data,
                       out["makespan_f32"].ctypes.data)


def _best_dict(b: _Best, st: int, ctx_ptr) -> dict:
    if st not in (OK, EINFEASIBLE):
        raise AdaptisError(st, _err(ctx_ptr))
    p = b.p
    return {"status": st, "index": int(b.index), "plan": plan_dict(b.plan),
            "makespan": int(b.result.makespan), "peak_mem": int(b.result.peak_mem_bytes),
            "makespan_f32": float(b.result.makespan_f32),
            "bubble": float(b.result.bubble_ratio), "throughput": float(b.result.throughput),
            "cand_status": int(b.result.status),
            "T_d": list(b.T_d[:p]), "busy_d": list(b.busy_d[:p]), "M_d": list(b.M_d[:p]),
            **{k: list(getattr(b, k)[:p]) for k in ACCT},
            "n_candidates": int(b.n_candidates), "n_evaluated": int(b.n_evaluated),
            "n_invalid": int(b.n_invalid), "n_tasks": int(b.n_tasks), "n_pruned": int(b.n_pruned),
            "kernel_ms": float(b.kernel_ms)}


def _device_int64_view(ptr: int, device: int):
    """A 1-element int64 torch tensor aliasing device memory at ptr."""
    import torch

    class _Holder:
        def __init__(self, p):
            self.__cuda_array_interface__ = {"shape": (1,), "typestr": "<i8", "data": (p, False),
                                             "version": 3}
    with torch.cuda.device(device):
        return torch.as_tensor(_Holder(ptr), device="cuda:%d" % device)
