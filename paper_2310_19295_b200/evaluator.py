"""Peak-memory evaluation on the GPU -- drop-ins for the reference's
``memplan.graph`` evaluators plus the batched candidate API.

Reference functions mirrored (pkg/src/memplan/graph.py):
  validate_schedule      375-398   -> rm_eval_schedule(RM_SCHED_VALIDATE)
  sequential_schedule    401-409
  tensor_lifetimes       440-449   -> rm_eval_schedule(birth/death)
  live_bytes_by_timestep 452-458   -> rm_eval_schedule(live)
  peak_memory            461-468   -> rm_eval_schedule(VALIDATE|PEAK)
New batched API:
  evaluate_orders(g, orders[B, n]) -> (peak i64[B], argmax i32[B], valid bool[B])
      elementwise peak_memory(g, sequential_schedule(g, o))        (K1)
  argmin_orders(...)  first strict minimum (tests/oracles.py:46-56)
  generate_orders(g, seed, first_id, B)  counter-RNG Kahn candidates on device
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .graph import ConfigError, Schedule, ScheduleError, graph_arrays, graph_cache


# ------------------------------------------------------------ graph handle

class DeviceGraph:
    """Owns an RmGraph handle (CSR + K1 metadata, host and device copies)."""

    def __init__(self, g, reduce: bool = True):
        a = graph_arrays(g)
        self.arrays = a
        self.n_ops, self.n_tensors = a.n_ops, a.n_tensors
        d = _lib.RmGraphDesc(a.n_ops, a.n_tensors, ptr(a.size), ptr(a.producer), ptr(a.cons_ptr),
                             ptr(a.cons_idx), ptr(a.in_ptr), ptr(a.in_idx), ptr(a.out_ptr),
                             ptr(a.out_idx))
        h = C.c_void_p()
        check(lib().rm_graph_create(C.byref(d), 0 if reduce else _lib.RM_NO_REDUCE, C.byref(h)),
              "rm_graph_create")
        self.handle = h.value
        self._destroy = lib().rm_graph_destroy

    def info(self) -> dict:
        inf = _lib.RmGraphInfo()
        check(lib().rm_graph_info(self.handle, C.byref(inf)), "rm_graph_info")
        return {f: getattr(inf, f) for f, _ in inf._fields_}

    def k1_export(self) -> dict:
        i = self.info()
        n = self.n_ops
        out = dict(
            vidx=np.empty(n, np.int32), slot=np.empty(n, np.int32),
            out_tab=np.empty(i["n_values"], np.int64), fs_tab=np.empty(i["n_values"], np.int64),
            edge_u=np.empty(i["n_check_edges"], np.int32), edge_v=np.empty(i["n_check_edges"], np.int32),
            mptr=np.empty(i["n_multi"] + 1, np.int32), mcons=np.empty(i["n_multi_cons"], np.int32),
            msize=np.empty(i["n_multi"], np.int64))
        check(lib().rm_graph_k1_export(self.handle, *(ptr(out[k]) for k in (
            "vidx", "slot", "out_tab", "fs_tab", "edge_u", "edge_v", "mptr", "mcons", "msize"))),
            "rm_graph_k1_export")
        return out

    def close(self) -> None:
        if self.handle:
            self._destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_graph(g) -> DeviceGraph:
    ent = graph_cache(g)
    dg = ent.get("device")
    if dg is None:
        dg = DeviceGraph(g)
        ent["device"] = dg
        ent["close"] = dg.close
    return dg


def _stream_handle(stream) -> int | None:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream or None
        except Exception:
            return None
        return None
    return getattr(stream, "cuda_stream", stream) or None


def _on(stream):
    """Allocate a call's outputs on the stream its kernels run on: torch's
    caching allocator ties a block to the stream current at allocation, so
    outputs made on another stream could be reused while the kernels still
    write them (a raw handle is the caller's to order)."""
    import contextlib
    if stream is not None and hasattr(stream, "cuda_stream"):
        import torch
        return torch.cuda.stream(stream)
    return contextlib.nullcontext()


# ------------------------------------------------------ single schedules

_MSG = {
    1: "schedule must contain every op exactly once",
    2: "timesteps must cover every op",
    4: "timesteps must be non-decreasing along the order",
}


def _as_i32(seq: Iterable[int]) -> np.ndarray:
    arr = np.asarray(tuple(seq), dtype=np.int64)
    if arr.size and (arr.min() < -(2**31) or arr.max() >= 2**31):
        raise ValueError("schedule values exceed int32")
    return arr.astype(np.int32)


def _run_schedule(g, s: Schedule, flags: int, want_spans: bool = False, want_live: bool = False):
    _lib.require_device()
    dg = device_graph(g)
    order = _as_i32(s.order)
    ts = _as_i32(s.timesteps)
    if len(ts) < dg.n_ops and not (flags & _lib.RM_SCHED_VALIDATE):
        raise IndexError("tuple index out of range")  # reference indexes s.timesteps[op]
    if ts.size and ts.min() < 0:
        raise ValueError("negative timesteps are not supported")
    steps = int(ts.max()) + 1 if ts.size else 0
    res = _lib.RmScheduleResult()
    birth = np.empty(dg.n_tensors, np.int32) if want_spans else None
    death = np.empty(dg.n_tensors, np.int32) if want_spans else None
    live = np.empty(max(steps, 1), np.int64) if want_live else None
    check(lib().rm_eval_schedule(dg.handle, ptr(order), len(order), ptr(ts), len(ts),
                                 int(s.ops_per_step), flags, C.byref(res), ptr(birth), ptr(death),
                                 ptr(live), None), "rm_eval_schedule")
    if res.status:
        if res.status == 3:
            raise ConfigError("ops_per_step must be >= 1")
        if res.status == 5:
            counts: dict[int, int] = {}
            for t in s.timesteps:  # message detail only (graph.py:390-394)
                counts[t] = counts.get(t, 0) + 1
                if counts[t] > s.ops_per_step:
                    raise ScheduleError(f"timestep {t} holds more than {s.ops_per_step} ops")
        if res.status == 6:
            raise ScheduleError(f"op {res.detail_a} scheduled before its predecessor {res.detail_b}")
        raise ScheduleError(_MSG[res.status])
    return res, birth, death, (live[:steps] if live is not None else None)


def validate_schedule(g, s: Schedule) -> None:
    """Raise ScheduleError/ConfigError unless s is valid (graph.py:375-398)."""
    _run_schedule(g, s, _lib.RM_SCHED_VALIDATE)


def sequential_schedule(g, order: Iterable[int], ops_per_step: int = 1) -> Schedule:
    """One op per timestep (graph.py:401-409); validated on the GPU."""
    order = tuple(order)
    ts = [0] * len(g.ops)
    for i, op in enumerate(order):
        ts[op] = i
    s = Schedule(order=order, timesteps=tuple(ts), ops_per_step=ops_per_step)
    validate_schedule(g, s)
    return s


def tensor_lifetimes(g, s: Schedule) -> list[tuple[int, int]]:
    """Per tensor inclusive [birth, death] (graph.py:440-449)."""
    _, b, d, _ = _run_schedule(g, s, 0, want_spans=True)
    return list(zip(b.tolist(), d.tolist()))


def live_bytes_by_timestep(g, s: Schedule) -> list[int]:
    """Live bytes per timestep (graph.py:452-458); no validation, like the reference."""
    _, _, _, live = _run_schedule(g, s, _lib.RM_SCHED_PEAK, want_live=True)
    return live.tolist()


def peak_memory(g, s: Schedule) -> tuple[int, int]:
    """(max live bytes, first timestep reaching it) (graph.py:461-468)."""
    res, _, _, _ = _run_schedule(g, s, _lib.RM_SCHED_VALIDATE | _lib.RM_SCHED_PEAK)
    if len(g.ops) == 0:
        return 0, 0
    return int(res.peak), int(res.argmax)


# ------------------------------------------------------- candidate batches

def _row_kind(orders):
    """('dev'|'host', flags) for an orders array: int32 rows, or uint16 rows
    (RM_ORDERS_U16: half the bytes to stage over PCIe and to read from HBM)."""
    if hasattr(orders, "is_cuda") and orders.is_cuda:
        import torch
        if orders.dtype == torch.int32:
            return "dev", _lib.RM_DEVICE_PTRS
        if orders.dtype == torch.uint16:
            return "dev", _lib.RM_DEVICE_PTRS | _lib.RM_ORDERS_U16
        raise ValueError("device orders must be int32 or uint16")
    return "host", 0


def _device_outputs(orders, B):
    import torch
    return (torch.empty(B, dtype=torch.int64, device=orders.device),
            torch.empty(B, dtype=torch.int32, device=orders.device),
            torch.empty(B, dtype=torch.uint8, device=orders.device))


def _host_rows(orders, n):
    """Host rows as a C-contiguous int32 or uint16 array (other integer
    types are checked and converted to int32; out-of-range ids become -1 so
    the row is reported invalid, as the reference would raise)."""
    if hasattr(orders, "numpy"):
        orders = orders.numpy()
    o = np.asarray(orders)
    if o.dtype in (np.int32, np.uint16) and o.ndim == 2 and o.shape[1] == n:
        return np.ascontiguousarray(o), (_lib.RM_ORDERS_U16 if o.dtype == np.uint16 else 0)
    o = np.ascontiguousarray(np.asarray(orders, dtype=np.int64))
    if o.ndim != 2 or o.shape[1] != n:
        if o.size == 0 and n == 0:
            o = o.reshape(-1, 0)
        else:
            raise ValueError(f"orders must be [B, {n}]")
    oor = (o < 0) | (o >= max(n, 1)) if o.size else np.zeros(o.shape, bool)
    return np.where(oor, -1, o).astype(np.int32), 0


def evaluate_orders(g, orders, stream=None):
    """Batched ``peak_memory(g, sequential_schedule(g, o))`` over rows of orders.

    ``orders``: [B, n_ops] host array-like (numpy; staged through the device
    inside the call) or a CUDA torch tensor (device path, async on
    ``stream``); int32 rows, or uint16 rows for graphs under 65,536 ops.
    Returns ``(peak int64[B], argmax int32[B], valid bool[B])`` of the same
    kind.  Invalid rows (not a topological permutation) have valid=False and
    unspecified peak/argmax; the reference raises for them.
    """
    dg = device_graph(g)
    n = dg.n_ops
    kind, flags = _row_kind(orders)
    if kind == "dev":
        import torch
        if orders.dim() != 2 or orders.shape[1] != n:
            raise ValueError(f"orders must be [B, {n}]")
        with _on(stream):
            orders = orders.contiguous()
            B = orders.shape[0]
            peak, arg, val = _device_outputs(orders, B)
            check(lib().rm_eval_orders(dg.handle, ptr(orders), B, flags, ptr(peak), ptr(arg), ptr(val),
                                       _stream_handle(stream)), "rm_eval_orders")
        return peak, arg, val.view(torch.bool)
    _lib.require_device()
    o, flags = _host_rows(orders, n)
    B = o.shape[0]
    peak = np.empty(B, np.int64)
    arg = np.empty(B, np.int32)
    val = np.empty(B, np.uint8)
    check(lib().rm_eval_orders(dg.handle, ptr(o), B, flags, ptr(peak), ptr(arg), ptr(val),
                               _stream_handle(stream)), "rm_eval_orders")
    return peak, arg, val.astype(bool)


def evaluate_live(g, orders, stream=None):
    """Batched ``live_bytes_by_timestep(g, sequential_schedule(g, o))``
    (graph.py:452-458) over rows of orders (rm_eval_live): ``(live int64[B,
    n], valid bool[B])`` of the input's kind (numpy for host rows, CUDA
    tensors for CUDA rows).  Rows with valid=False have unspecified live
    values (the reference raises for them)."""
    dg = device_graph(g)
    n = dg.n_ops
    kind, flags = _row_kind(orders)
    if kind == "dev":
        import torch
        if orders.dim() != 2 or orders.shape[1] != n:
            raise ValueError(f"orders must be [B, {n}]")
        with _on(stream):
            orders = orders.contiguous()
            B = orders.shape[0]
            live = torch.empty((B, n), dtype=torch.int64, device=orders.device)
            val = torch.empty(B, dtype=torch.uint8, device=orders.device)
            check(lib().rm_eval_live(dg.handle, ptr(orders), B, flags, ptr(live), ptr(val),
                                     _stream_handle(stream)), "rm_eval_live")
        return live, val.view(torch.bool)
    _lib.require_device()
    o, flags = _host_rows(orders, n)
    B = o.shape[0]
    live = np.empty((B, n), np.int64)
    val = np.empty(B, np.uint8)
    check(lib().rm_eval_live(dg.handle, ptr(o), B, flags, ptr(live), ptr(val), _stream_handle(stream)),
          "rm_eval_live")
    return live, val.astype(bool)


def evaluate_and_select(g, orders, id_base: int = 0, stream=None):
    """evaluate_orders + first-strict-minimum selection in one libroam call
    (rm_eval_select).  Returns (peak, argmax, valid, best) where best is a
    (peak, id + id_base) pair -- a 2-element int64 CUDA tensor for device
    inputs (no host sync), a tuple for host inputs."""
    dg = device_graph(g)
    n = dg.n_ops
    kind, flags = _row_kind(orders)
    if kind == "dev":
        import torch
        if orders.dim() != 2 or orders.shape[1] != n:
            raise ValueError(f"orders must be [B, {n}]")
        with _on(stream):
            orders = orders.contiguous()
            B = orders.shape[0]
            peak, arg, val = _device_outputs(orders, B)
            best = torch.empty(2, dtype=torch.int64, device=orders.device)
            check(lib().rm_eval_select(dg.handle, ptr(orders), B, id_base, flags, ptr(peak), ptr(arg),
                                       ptr(val), ptr(best), _stream_handle(stream)), "rm_eval_select")
        return peak, arg, val, best
    _lib.require_device()
    o, flags = _host_rows(orders, n)
    B = o.shape[0]
    peak = np.empty(B, np.int64)
    arg = np.empty(B, np.int32)
    val = np.empty(B, np.uint8)
    best = np.empty(2, np.int64)
    check(lib().rm_eval_select(dg.handle, ptr(o), B, id_base, flags, ptr(peak), ptr(arg), ptr(val),
                               ptr(best), _stream_handle(stream)), "rm_eval_select")
    return peak, arg, val.astype(bool), (int(best[0]), int(best[1]))


def select_device(peak, valid, id_base: int = 0, stream=None):
    """Device-resident argmin: 2-element int64 CUDA tensor {peak, id + id_base}
    (no host synchronisation; the multi-GPU exchange consumes it directly)."""
    import torch
    with _on(stream):
        out = torch.empty(2, dtype=torch.int64, device=peak.device)
        v = valid.view(torch.uint8) if valid.dtype == torch.bool else valid.to(torch.uint8)
        check(lib().rm_argmin(ptr(peak), ptr(v), peak.shape[0], id_base, _lib.RM_DEVICE_PTRS, ptr(out),
                              _stream_handle(stream)), "rm_argmin")
    return out


def select_key_device(g, peak, valid, id_base: int, id_bits: int, stream=None):
    """Device-resident packed key (peak << id_bits) | id of the first strict
    minimum (INT64_MAX if none valid): one int64 for all_reduce(MIN)."""
    import torch
    with _on(stream):
        out = torch.empty(1, dtype=torch.int64, device=peak.device)
        v = valid.view(torch.uint8) if valid.dtype == torch.bool else valid.to(torch.uint8)
        check(lib().rm_argmin_key(ptr(peak), ptr(v), peak.shape[0], id_base, id_bits,
                                  device_graph(g).info()["total_bytes"], ptr(out), _stream_handle(stream)),
              "rm_argmin_key")
    return out


def evaluate_select_key(g, orders, id_base: int, id_bits: int, stream=None):
    """K1 over device rows with the packed-key selection fused into the same
    launch (rm_eval_select_key): (peak, argmax, valid, key) CUDA tensors, key
    = (peak << id_bits) | (id + id_base) of the first strict minimum, INT64_MAX
    if no row is valid -- select_key_device(evaluate_orders(...)) in one pass."""
    import torch
    dg = device_graph(g)
    n = dg.n_ops
    kind, flags = _row_kind(orders)
    if kind != "dev":
        raise ValueError("evaluate_select_key takes CUDA rows")
    if orders.dim() != 2 or orders.shape[1] != n:
        raise ValueError(f"orders must be [B, {n}]")
    with _on(stream):
        orders = orders.contiguous()
        B = orders.shape[0]
        peak, arg, val = _device_outputs(orders, B)
        key = torch.empty(1, dtype=torch.int64, device=orders.device)
        check(lib().rm_eval_select_key(dg.handle, ptr(orders), B, id_base, id_bits, flags, ptr(peak),
                                       ptr(arg), ptr(val), ptr(key), _stream_handle(stream)),
              "rm_eval_select_key")
    return peak, arg, val.view(torch.bool), key


def argmin_orders(peak, valid, id_base: int = 0, stream=None) -> tuple[int, int]:
    """First strict minimum (lexicographic (peak, id)) over valid candidates.

    Returns (peak, id + id_base), or (INT64_MAX, -1) if none is valid."""
    out = np.empty(2, np.int64)
    if hasattr(peak, "is_cuda") and peak.is_cuda:
        import torch
        with _on(stream):
            dout = torch.empty(2, dtype=torch.int64, device=peak.device)
            v = valid.view(torch.uint8) if valid.dtype == torch.bool else valid.to(torch.uint8)
            check(lib().rm_argmin(ptr(peak), ptr(v), peak.shape[0], id_base, _lib.RM_DEVICE_PTRS,
                                  ptr(dout), _stream_handle(stream)), "rm_argmin")
        return tuple(int(x) for x in dout.cpu().tolist())
    p = np.ascontiguousarray(peak, dtype=np.int64)
    v = np.ascontiguousarray(valid, dtype=np.uint8)
    check(lib().rm_argmin(ptr(p), ptr(v), len(p), id_base, 0, ptr(out), None), "rm_argmin")
    return int(out[0]), int(out[1])


def generate_orders(g, seed: int, first_id: int, B: int, device=None, stream=None):
    """Counter-RNG Kahn candidates materialised in HBM (int32[B, n] torch tensor)."""
    import torch
    dg = device_graph(g)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    with _on(stream):
        out = torch.empty((B, dg.n_ops), dtype=torch.int32, device=dev)
        check(lib().rm_gen_orders(dg.handle, seed & (2**64 - 1), first_id, B, ptr(out),
                                  _stream_handle(stream)), "rm_gen_orders")
    return out


def set_kernel_timing(enable: bool) -> None:
    lib().rm_set_timing(1 if enable else 0)


def asap_alap(g) -> tuple[tuple[int, ...], tuple[int, ...]]:
    """Schedule bounds (graph.py:365-372) from closure bitsets in libroam's
    C++ host code: (asap, alap) tuples, computed once per graph (the planner
    asks from the tree build and from weight-update placement)."""
    ent = graph_cache(g)
    hit = ent.get("asap_alap")
    if hit is None:
        dg = device_graph(g)
        n = dg.n_ops
        asap = np.zeros(n, np.int32)
        alap = np.zeros(n, np.int32)
        check(lib().rm_graph_asap_alap(dg.handle, ptr(asap), ptr(alap)), "rm_graph_asap_alap")
        hit = ent["asap_alap"] = (tuple(asap.tolist()), tuple(alap.tolist()))
    return hit


def set_sm_reserve(sms: int) -> None:
    """K1 leaves ``sms`` SMs idle (rm_set_sm_reserve), for a collective that
    overlaps the next batch's evaluation on another stream."""
    check(lib().rm_set_sm_reserve(int(sms)), "rm_set_sm_reserve")


def set_gen_form(form: int) -> None:
    """Candidate generator form on this thread: 0 auto (thread per candidate
    where the graph qualifies), 1 warp per candidate (rm_set_gen_form)."""
    check(lib().rm_set_gen_form(int(form)), "rm_set_gen_form")


def set_k1_variant(variant: int) -> None:
    """0 auto, 1 generic evaluator, 2 unit-packed interleaved (v2); per thread."""
    check(lib().rm_set_k1_variant(int(variant)), "rm_set_k1_variant")


def last_kernel_ms() -> float:
    return float(lib().rm_last_kernel_ms())


def launch_count() -> int:
    return int(lib().rm_launch_count())
