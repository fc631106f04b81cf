"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/peak_oracle.c (C restatement of the reference's
peak_memory over sequential orders, graph.py:375-468), multithreaded over
candidates.  Used by tests as the large-batch checker and by bench.py as the
CPU baseline / reference arm.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


def build() -> Path:
    src = HERE / "peak_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(LIB))
        _lib.oracle_eval_orders.restype = C.c_int
        _lib.oracle_eval_orders.argtypes = [C.c_int, C.c_int] + [C.c_void_p] * 7 + [
            C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.oracle_eval_orders_events.restype = C.c_int
        _lib.oracle_eval_orders_events.argtypes = _lib.oracle_eval_orders.argtypes
        _lib.oracle_kahn_orders.restype = C.c_int
        _lib.oracle_kahn_orders.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                            C.c_int64, C.c_int64, C.c_int, C.c_void_p]
    return _lib


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


class CGraph:
    """Flat arrays of a reference-shaped graph for the C oracle."""

    def __init__(self, g):
        self.n, self.T = len(g.ops), len(g.tensors)
        self.size = np.array([t.size for t in g.tensors], np.int64)
        self.producer = np.array([t.producer for t in g.tensors], np.int32)
        cl = [len(t.consumers) for t in g.tensors]
        self.cons_ptr = np.zeros(self.T + 1, np.int32)
        self.cons_ptr[1:] = np.cumsum(cl)
        self.cons_idx = np.array([c for t in g.tensors for c in t.consumers], np.int32)
        preds = []
        for op in g.ops:  # graph.py:97-104
            p = {g.tensors[t].producer for t in op.inputs}
            p.discard(op.id)
            preds.append(sorted(p))
        self.pred_ptr = np.zeros(self.n + 1, np.int32)
        self.pred_ptr[1:] = np.cumsum([len(p) for p in preds])
        self.pred_idx = np.array([q for p in preds for q in p], np.int32)
        succs = [[] for _ in range(self.n)]
        for v, p in enumerate(preds):
            for q in p:
                succs[q].append(v)
        self.succ_ptr = np.zeros(self.n + 1, np.int32)
        self.succ_ptr[1:] = np.cumsum([len(s) for s in succs])
        self.succ_idx = np.array([w for s in succs for w in s], np.int32)


def eval_orders(cg: CGraph, orders: np.ndarray, threads: int | None = None, events: bool = False):
    """(peak int64[B], argmax int32[B], valid bool[B]); invalid rows peak 0.
    events=True: lifetimes as a +size/-size event sweep (same results, O(n+T+E)
    per row) for checking million-row batches; the default keeps the
    reference's per-step add loop (graph.py:452-458)."""
    L = _load()
    o = np.ascontiguousarray(orders, dtype=np.int32)
    B = o.shape[0]
    peak = np.empty(B, np.int64)
    arg = np.empty(B, np.int32)
    val = np.empty(B, np.uint8)
    fn = L.oracle_eval_orders_events if events else L.oracle_eval_orders
    fn(cg.n, cg.T, _p(cg.size), _p(cg.producer), _p(cg.cons_ptr), _p(cg.cons_idx),
                         _p(cg.pred_ptr), _p(cg.pred_idx), _p(o), B, threads or os.cpu_count() or 1,
                         _p(peak), _p(arg), _p(val))
    return peak, arg, val.astype(bool)


def kahn_orders(cg: CGraph, seed: int, first_id: int, B: int, threads: int | None = None) -> np.ndarray:
    """Counter-RNG Kahn candidates (same rows as memplan_oracle.kahn_candidate)."""
    L = _load()
    out = np.empty((B, cg.n), np.int32)
    L.oracle_kahn_orders(cg.n, _p(cg.pred_ptr), _p(cg.succ_ptr), _p(cg.succ_idx), seed & (2**64 - 1),
                         first_id, B, threads or os.cpu_count() or 1, _p(out))
    return out
