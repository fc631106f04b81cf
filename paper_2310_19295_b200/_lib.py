"""Build and load ``libroam.so`` -- the C-ABI library declared in
``include/roam.h`` (sm_100a kernels + host-side graph marshalling).

The shared object is built in-tree (``paper_2310_19295_b200/libroam.so``) with
nvcc directly, so it travels with the repo snapshot to the GPU box.  There is
no CPU fallback anywhere: if the library or a CUDA device is missing the
product API raises.
"""

from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_PATH = PKG / "libroam.so"
SOURCES = ("roam_graph.cpp", "layout_search.cpp", "order_search.cpp", "wu_place.cpp", "nccl_select.cpp", "k_eval.cu", "k_eval_v4.cu", "k_eval_v5.cu", "k_gen.cu", "k_layout.cu", "k_repair.cu", "k_live.cu", "k_pack.cu", "k_greedy.cu", "k_exact.cu")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


class RoamError(RuntimeError):
    """A libroam call failed (status code + rm_last_error message)."""


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RoamError("nvcc not found: cannot build libroam")


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every translation unit for sm_100a and link libroam.so."""
    srcs = [CSRC / s for s in SOURCES]
    deps = srcs + [CSRC / "roam_internal.h", CSRC / "k_common.cuh", ROOT / "include" / "roam.h"]
    if not force and LIB_PATH.exists():
        newest = max(p.stat().st_mtime for p in deps)
        if LIB_PATH.stat().st_mtime >= newest:
            return LIB_PATH
    nvcc = _nvcc()
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    common = [nvcc, "-std=c++17", "-O3", ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O3,-mpopcnt",
              "-I", str(ROOT / "include")]

    hdr_t = max(p.stat().st_mtime for p in deps[len(srcs):])

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.name + ".o")
        # an object newer than its source and every header is reused
        if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_t):
            return obj
        cmd = common + ["-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RoamError(f"nvcc failed on {src.name}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = LIB_PATH.with_suffix(".so.tmp")
    r = subprocess.run([nvcc, ARCH, "-shared", "-o", str(tmp)] + [str(o) for o in objs] + ["-ldl"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RoamError(f"nvcc link failed:\n{r.stderr}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


# ----------------------------------------------------------------- ctypes

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p


class RmGraphDesc(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("n_tensors", C.c_int32),
                ("size", vp), ("producer", vp), ("cons_ptr", vp), ("cons_idx", vp),
                ("in_ptr", vp), ("in_idx", vp), ("out_ptr", vp), ("out_idx", vp)]


class RmGraphInfo(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("n_tensors", C.c_int32), ("n_cons", C.c_int64),
                ("n_pred_edges", C.c_int64), ("n_check_edges", C.c_int64),
                ("n_multi", C.c_int64), ("n_multi_cons", C.c_int64), ("n_slots", C.c_int64),
                ("n_values", C.c_int64), ("reduced", C.c_int32), ("wide_index", C.c_int32),
                ("total_bytes", C.c_int64), ("k1_variant", C.c_int32), ("unit_shift", C.c_int32)]


class RmScheduleResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("detail_a", C.c_int32), ("detail_b", C.c_int32),
                ("n_steps", C.c_int32), ("peak", C.c_int64), ("argmax", C.c_int32),
                ("_pad", C.c_int32)]


RM_ERR_CAPACITY = -5
RM_ERR_GRAPH = -6
RM_DEVICE_PTRS = 1
RM_NO_REDUCE = 2
RM_ORDERS_U16 = 4
RM_SCHED_VALIDATE = 1 << 8
RM_SCHED_PEAK = 1 << 9
RM_LLFB_PLAIN, RM_LLFB_CONSTRAINED, RM_LLFB_COMPONENTS = 0, 1, 2

# name -> (restype, argtypes); every symbol include/roam.h declares
SIGNATURES = {
    "rm_graph_create": (C.c_int, [C.POINTER(RmGraphDesc), C.c_uint32, C.POINTER(vp)]),
    "rm_graph_destroy": (C.c_int, [vp]),
    "rm_graph_info": (C.c_int, [vp, C.POINTER(RmGraphInfo)]),
    "rm_graph_k1_export": (C.c_int, [vp] + [vp] * 9),
    "rm_eval_orders": (C.c_int, [vp, vp, C.c_int64, C.c_uint32, vp, vp, vp, vp]),
    "rm_eval_select": (C.c_int, [vp, vp, C.c_int64, C.c_int64, C.c_uint32, vp, vp, vp, vp, vp]),
    "rm_argmin": (C.c_int, [vp, vp, C.c_int64, C.c_int64, C.c_uint32, vp, vp]),
    "rm_argmin_key": (C.c_int, [vp, vp, C.c_int64, C.c_int64, C.c_int32, C.c_int64, vp, vp]),
    "rm_gen_orders": (C.c_int, [vp, C.c_uint64, C.c_int64, C.c_int64, vp, vp]),
    "rm_eval_schedule": (C.c_int, [vp, vp, C.c_int64, vp, C.c_int64, C.c_int32, C.c_uint32,
                                   C.POINTER(RmScheduleResult), vp, vp, vp, vp]),
    "rm_layout_violations": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp, C.c_int64, vp, vp,
                                       C.c_int64, vp, vp, vp]),
    "rm_repair_place": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp, vp, C.c_int64, vp]),
    "rm_repair_conflicts": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "rm_place_weight_updates": (C.c_int, [C.c_int32, vp, C.c_int64, vp, vp, vp, C.c_double, C.c_int32, vp, vp,
                                          C.c_int32, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp,
                                          C.c_double, C.c_int32] + [vp] * 8),
    "rm_llfb_batch": (C.c_int, [C.c_int32, vp, vp, vp, vp, vp, vp, C.c_int32, vp, vp, vp, vp,
                                vp, vp]),
    "rm_layout_search": (C.c_int, [C.c_int32, vp, vp, vp, vp, vp, C.c_int32, vp, C.c_int64, C.c_double,
                                   vp, vp, vp, vp]),
    "rm_exact_order_search": (C.c_int, [vp, C.c_int32, vp, C.c_int64, vp, C.c_int64, vp, C.c_int64,
                                        C.c_double, vp, vp, vp, vp, vp]),
    "rm_greedy_windows": (C.c_int, [vp, C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "rm_exact_windows": (C.c_int, [vp, C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "rm_last_error": (C.c_char_p, []),
    "rm_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "rm_launch_count": (C.c_int64, []),
    "rm_set_timing": (C.c_int, [C.c_int]),
    "rm_set_k1_variant": (C.c_int, [C.c_int]),
    "rm_set_sm_reserve": (C.c_int, [C.c_int]),
    "rm_set_gen_form": (C.c_int, [C.c_int]),
    "rm_set_pack_form": (C.c_int, [C.c_int]),
    "rm_nccl_unique_id": (C.c_int, [vp, C.c_int64]),
    "rm_nccl_comm_init": (C.c_int, [C.c_int32, vp, C.c_int32, C.POINTER(vp)]),
    "rm_nccl_comm_destroy": (C.c_int, [vp]),
    "rm_nccl_select_key": (C.c_int, [vp, vp, vp]),
    "rm_graph_asap_alap": (C.c_int, [vp, vp, vp]),
    "rm_graph_ancestors": (C.c_int, [vp, vp]),
    "rm_popcount_rows": (C.c_int, [vp, C.c_int64, C.c_int64, vp, vp]),
    "rm_eval_live": (C.c_int, [vp, vp, C.c_int64, C.c_uint32, vp, vp, vp]),
    "rm_eval_select_key": (C.c_int, [vp, vp, C.c_int64, C.c_int64, C.c_int32, C.c_uint32, vp, vp, vp, vp, vp]),
    "rm_last_kernel_ms": (C.c_double, []),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """The loaded libroam (built on first use if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                build()
            L = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = lib().rm_last_error().decode(errors="replace")
        raise RoamError(f"{what or 'libroam'} failed (status {status}): {msg}")


def device_count() -> int:
    c = C.c_int(0)
    check(lib().rm_device_count(C.byref(c)), "rm_device_count")
    return c.value


def require_device() -> None:
    if device_count() == 0:
        raise RoamError("no CUDA device visible: the ROAM B200 path has no CPU fallback")


def ptr(a) -> int | None:
    """Address of a numpy array / torch tensor buffer (None for empty)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr() or None
    return a.ctypes.data if a.size else None
