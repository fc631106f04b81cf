"""Candidate sharding across GPUs and the global (peak, id) argmin.

Candidates are independent units: rank r of W evaluates the
contiguous id range [r*B/W, (r+1)*B/W) of a candidate batch, with no data-path
collective; the only exchange is one all_gather of each rank's 16-byte best
{peak:int64, id:int64}.  The lexicographic min of (peak, id) over the gathered
pairs equals the reference's first strict minimum over the global id order
(tests/oracles.py:46-56 ``peak < best``; planner.py:209-216), because ids are
globally unique and ranks own disjoint ranges.

One process per GPU; ``torch.distributed`` carries the exchange (NCCL over
NVLink on the GPU box, gloo in the CPU tests).  Graph metadata is replicated:
every rank builds the same graph and its own device handle.
"""

from __future__ import annotations

from dataclasses import dataclass

NONE_PEAK = 2**63 - 1


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) candidate ids of ``rank``: contiguous, sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def lex_min(pairs) -> tuple[int, int]:
    """Lexicographic min of (peak, id) pairs, ignoring id == -1 (no valid
    candidate on that rank); (INT64_MAX, -1) when none is valid."""
    best = (NONE_PEAK, -1)
    for peak, cid in pairs:
        peak, cid = int(peak), int(cid)
        if cid < 0:
            continue
        if best[1] < 0 or (peak, cid) < best:
            best = (peak, cid)
    return best


def allgather_best(best, group=None):
    """Exchange each rank's best {peak, id} (int64[2] tensor on the rank's
    device for NCCL, on CPU for gloo) and return the global lexicographic min
    as a tensor of the same kind (every rank gets the same answer)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = best.device
    if dist.get_backend(group) == "gloo" and dev.type == "cuda":
        best = best.cpu()  # gloo gathers host tensors (CPU tests / shared-GPU runs)
    out = torch.empty(world * 2, dtype=torch.int64, device=best.device)
    dist.all_gather_into_tensor(out, best.contiguous(), group=group)
    out = out.to(dev)
    pk = out.view(world, 2)
    big = torch.full_like(pk[:, 0], NONE_PEAK)
    ids = torch.where(pk[:, 1] < 0, big, pk[:, 1])   # ranks with nothing valid lose
    m = pk[:, 0].min()
    idmin = torch.where(pk[:, 0] == m, ids, big).min()
    return torch.stack([m, torch.where(idmin == NONE_PEAK, torch.full_like(idmin, -1), idmin)])


def key_bits(total_candidates: int) -> int:
    """id bits of the packed (peak << bits) | id key for ids < total."""
    return max(1, (max(total_candidates, 1) - 1).bit_length())


def allreduce_key(key, group=None):
    """One all_reduce(MIN) of the 8-byte packed key: the global first strict
    minimum (lexicographic (peak, id), since ids fit below the peak bits)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "gloo" and key.device.type == "cuda":
        k = key.cpu()
        dist.all_reduce(k, op=dist.ReduceOp.MIN, group=group)
        key.copy_(k)
    else:
        dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    return key


def decode_key(key: int, bits: int) -> tuple[int, int]:
    return (NONE_PEAK, -1) if key == NONE_PEAK else (key >> bits, key & ((1 << bits) - 1))


@dataclass(frozen=True)
class ShardResult:
    best_peak: int
    best_id: int
    local_range: tuple[int, int]
    local_valid: int


def evaluate_sharded(g, total: int, seed: int = 0, group=None, stream=None,
                     chunk: int = 1 << 16) -> ShardResult:
    """Generate this rank's candidate ids on its device (counter-RNG Kahn),
    evaluate them with K1 and keep the first strict minimum on the device,
    ``chunk`` candidates at a time (rows never exceed chunk x n in HBM), then
    exchange it: the 8-GPU candidate search of BASELINE config 5."""
    import torch
    import torch.distributed as dist

    from . import evaluator as ev
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(total, world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    # every allocation and torch op of the loop on the kernels' stream
    with ev._on(stream):
        best = torch.tensor([NONE_PEAK, -1], dtype=torch.int64, device=dev)
        n_valid = torch.zeros((), dtype=torch.int64, device=dev)
        for c0 in range(lo, hi, max(1, chunk)):
            nb = min(chunk, hi - c0)
            orders = ev.generate_orders(g, seed, c0, nb, device=dev, stream=stream)
            peak, _, valid = ev.evaluate_orders(g, orders, stream=stream)
            cb = ev.select_device(peak, valid, id_base=c0, stream=stream)
            n_valid += valid.sum()
            # chunks arrive in id order: a later chunk wins only with a strictly smaller peak
            take = (cb[1] >= 0) & ((best[1] < 0) | (cb[0] < best[0]))
            best = torch.where(take, cb, best)
    if stream is not None and hasattr(stream, "synchronize"):
        torch.cuda.current_stream().wait_stream(stream)
    if world > 1:
        best = allgather_best(best, group)
    b = [int(x) for x in best.cpu().tolist()]
    return ShardResult(b[0], b[1], (lo, hi), int(n_valid.item()))


class NcclSelect:
    """libroam's own selection exchange (rm_nccl_select_key): an NCCL
    communicator over the ranks and one 8-byte ncclAllReduce(MIN) of each
    rank's packed key, for hosts that do not run torch.distributed (the
    C-ABI path a C/C++ planner host binds).  ``uid`` is rank 0's
    ``NcclSelect.unique_id()``, shipped to the other ranks out of band."""

    def __init__(self, nranks: int, uid: bytes, rank: int):
        import ctypes as C

        from ._lib import check, lib
        self._lib = lib()
        buf = (C.c_uint8 * len(uid)).from_buffer_copy(uid)
        comm = C.c_void_p()
        check(self._lib.rm_nccl_comm_init(int(nranks), buf, int(rank), C.byref(comm)), "rm_nccl_comm_init")
        self.comm = comm

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C

        from ._lib import check, lib
        buf = (C.c_uint8 * 128)()
        check(lib().rm_nccl_unique_id(buf, 128), "rm_nccl_unique_id")
        return bytes(buf)

    def select(self, key, stream=None):
        """In place: key (device int64[1]) <- the min over the ranks' keys."""
        from ._lib import check
        from .evaluator import _stream_handle
        check(self._lib.rm_nccl_select_key(self.comm, key.data_ptr(), _stream_handle(stream)),
              "rm_nccl_select_key")
        return key

    def close(self):
        from ._lib import check
        if self.comm:
            check(self._lib.rm_nccl_comm_destroy(self.comm), "rm_nccl_comm_destroy")
            self.comm = None
