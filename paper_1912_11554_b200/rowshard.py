"""Row sharding of one logistic-regression chain across GPUs.

SURVEY.md 8(e), BASELINE config 5 (8M x 255, one chain): the reference
evaluates the potential and gradient (kernels.py:90-123) over all N rows in
one process.  Here rank g of `world` holds rows ``row_range(N, g, world)``
and every rank runs the SAME chain (same keys, same calls).  Inside the
persistent kernel, each data pass ends with an exchange over NVLink peer
memory (csrc/ts_logistic.cuh, logistic_eval_grid): every GPU pushes its
exact fixed-point totals (p + 2 values as int64 pairs) into every peer's
mailbox and adds the `world` copies it receives.  Integer addition is
order-free, so all ranks see identical U and gradients -- bit-identical to
one GPU holding all rows -- and take identical tree decisions.

Host plumbing only: the mailboxes are cudaMalloc'd by the library, their
CUDA IPC handles are all-gathered by the caller (``torch_all_gather`` over
torch.distributed, any backend), and the library maps the peers.
"""

from __future__ import annotations

import ctypes
from typing import Callable, List, Sequence, Tuple

import numpy as np

from . import _lib

HANDLE_BYTES = 64
MAX_PEERS = 8


TILE_ROWS = 32  # rows per exact-accumulation group of the wide (64 < p <= 256) pass


def row_range(n_rows: int, rank: int, world: int, align: int = TILE_ROWS) -> Tuple[int, int]:
    """Rows [start, stop) of rank `rank`: contiguous, whole `align`-row tiles
    (so every rank's tiles are exactly the single-GPU tiles), tile counts
    differing by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank/world out of range")
    tiles = -(-n_rows // align)
    t0, t1 = (rank * tiles) // world, ((rank + 1) * tiles) // world
    return min(n_rows, t0 * align), min(n_rows, t1 * align)


def torch_all_gather(group=None) -> Callable[[bytes], List[bytes]]:
    """An all-gather of small byte strings over torch.distributed (rank order)."""
    import torch.distributed as dist

    def gather(b: bytes) -> List[bytes]:
        out: list = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, b, group=group)
        return out

    return gather


def connect(spec, rank: int, world: int, all_gather: Callable[[bytes], Sequence[bytes]], device=None) -> None:
    """Join this rank's logistic model (built from its row shard) to the
    row-sharded group.  Collective: every rank calls it once, in any order.
    ``spec`` is the model's DeviceSpec; ``all_gather(bytes) -> [bytes]*world``."""
    if spec.kind != _lib.TS_LOGISTIC:
        raise ValueError("row sharding applies to logistic_regression models")
    if not 1 <= world <= MAX_PEERS or not 0 <= rank < world:
        raise ValueError(f"world must be in [1, {MAX_PEERS}] and 0 <= rank < world")
    lib = _lib.load_library()
    h = spec.handle(device)
    buf = ctypes.create_string_buffer(HANDLE_BYTES)
    _lib.check(lib.ts_peer_mailbox_create(h, rank, world, buf))
    handles = list(all_gather(bytes(buf.raw)))
    if len(handles) != world or any(len(x) != HANDLE_BYTES for x in handles):
        raise RuntimeError("row-shard handle exchange returned a malformed list")
    joined = ctypes.create_string_buffer(b"".join(handles), HANDLE_BYTES * world)
    _lib.check(lib.ts_peer_mailbox_connect(h, joined))
    spec.row_shard = (rank, world)


def emulate_ranks(spec, vranks: int, device=None) -> None:
    """Test mode: run `vranks` row-sharded ranks inside ONE cooperative launch
    on one GPU (groups of CTAs with their own rows, barriers and accumulators,
    exchanging through the same mailbox device code as connect()).  The
    wide-p model's chain is then bit-identical to the unsharded run."""
    lib = _lib.load_library()
    _lib.check(lib.ts_model_set_virtual_ranks(spec.handle(device), int(vranks)))


# ----------------------------------------------------------------------------- fixed-point totals


def partial_sums(spec, q, device=None) -> np.ndarray:
    """Raw fixed-point totals of one evaluation at q over this model's rows
    (before any exchange): uint64[2*(p+2)+1] (ts_logistic_partial_sums)."""
    torch = _lib.torch_cuda()
    dev = _lib.cuda_device(torch, device)
    lib = _lib.load_library()
    h = spec.handle(dev)
    p = spec.dim - 1
    qd = torch.from_numpy(np.ascontiguousarray(q, dtype=np.float64)).to(dev)
    words = torch.zeros(2 * (p + 2) + 1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(lib.ts_logistic_partial_sums(h, _lib.ptr(qd), _lib.ptr(words), _lib.stream_ptr(torch)))
        torch.cuda.synchronize(dev)
    return words.cpu().numpy().view(np.uint64).copy()


LO_BITS = 51  # fixed-point pair: value = hi * 2^-10 + lo * 2^-61 (csrc fx_split)


def canonical(hi, lo):
    """(hi, lo) uint64 words -> canonical pair with lo in [0, 2^51) (csrc fx_canon)."""
    hi = np.asarray(hi, dtype=np.uint64)
    lo = np.asarray(lo, dtype=np.uint64)
    with np.errstate(over="ignore"):
        hi = hi + (lo.view(np.int64) >> np.int64(LO_BITS)).view(np.uint64)
    return hi, lo & np.uint64((1 << LO_BITS) - 1)


def combine(words_per_rank: Sequence[np.ndarray]) -> np.ndarray:
    """Wrapping uint64 sum of the ranks' totals -- what every GPU computes."""
    acc = np.zeros_like(np.asarray(words_per_rank[0], dtype=np.uint64))
    with np.errstate(over="ignore"):
        for w in words_per_rank:
            acc = acc + np.asarray(w, dtype=np.uint64)
    return acc


def totals_to_potential_gradient(words: np.ndarray, q) -> np.ndarray:
    """(U, gradient) from combined totals, the device's own arithmetic
    (fx_canon + fx_join, prior 0.5|q|^2 summed bias first, g = q - s)."""
    q = np.asarray(q, dtype=np.float64)
    p = q.size - 1
    w = np.asarray(words, dtype=np.uint64)
    if w[2 * (p + 2)] != 0:
        s = np.full(p + 2, np.nan)
    else:
        hi_u, lo_u = canonical(w[0:2 * (p + 2):2], w[1:2 * (p + 2):2])
        hi = hi_u.view(np.int64).astype(np.float64)
        lo = lo_u.astype(np.float64)
        s = hi * (1.0 / 1024.0) + lo * (1.0 / 2305843009213693952.0)
    prior = 0.5 * q[p] * q[p]
    for d in range(p):
        prior += 0.5 * q[d] * q[d]
    out = np.empty(p + 2)
    out[0] = prior - s[p + 1]
    out[1:] = q - s[:p + 1]
    return out
