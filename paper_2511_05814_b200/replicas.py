"""Independent decode replicas, one engine per GPU ("replicas only").

Routing and caches never interact across GPUs, so the hot path has no collective; the only
cross-rank traffic is the bench's timing reduction.  What ranks of one node do share is the
host expert store: 90 GB (8x7B) or 271 GB (8x22B) per copy does not fit once per GPU in host
DRAM, so local rank 0 creates a POSIX shared-memory segment, fills it, and every local rank's
engine page-locks the same pages (moe_engine_create_ex).  The experts are the model's weights,
identical for every replica; each replica serves its own request stream.
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass
from multiprocessing import shared_memory
from typing import Callable, Optional

TOKENS_PER_RANK_STREAM = 1_000_000  # token-id offset between replicas' synthetic streams


def rank_token_base(rank: int) -> int:
    """First synthetic token index of a replica's request stream (streams never overlap)."""
    return rank * TOKENS_PER_RANK_STREAM


def store_name(config, seed: int, job: str = "") -> str:
    """Deterministic shm name for a model shape + seed (+ job id, to isolate concurrent jobs)."""
    key = f"{config.num_layers}x{config.num_experts}x{config.hidden_dim}x{config.ffn_dim}:" \
          f"{config.expert_kind}:{seed}:{job}"
    return "moeb200_" + hashlib.sha1(key.encode()).hexdigest()[:16]


@dataclass
class SharedExpertStore:
    """A named host memory segment holding [L][E][expert] bytes."""

    shm: shared_memory.SharedMemory
    owner: bool

    @classmethod
    def create(cls, name: str, nbytes: int) -> "SharedExpertStore":
        try:  # a stale segment from a killed run
            old = shared_memory.SharedMemory(name=name)
            old.close()
            old.unlink()
        except FileNotFoundError:
            pass
        return cls(shared_memory.SharedMemory(name=name, create=True, size=nbytes), True)

    @classmethod
    def attach(cls, name: str) -> "SharedExpertStore":
        shm = shared_memory.SharedMemory(name=name)
        # Python < 3.13 registers attached segments with this process's resource tracker,
        # which would unlink the owner's segment when an attaching replica exits first
        from multiprocessing import resource_tracker

        try:
            resource_tracker.unregister(shm._name, "shared_memory")
        except Exception:
            pass
        return cls(shm, False)

    @property
    def nbytes(self) -> int:
        return self.shm.size

    @property
    def address(self) -> int:
        import ctypes

        return ctypes.addressof(ctypes.c_char.from_buffer(self.shm.buf))

    def close(self) -> None:
        try:
            self.shm.close()
        except BufferError:  # a ctypes view still alive: the mapping dies with the process
            pass
        if self.owner:
            try:
                self.shm.unlink()
            except FileNotFoundError:
                pass


def parse_node_list(text: str) -> list:
    """'0-1,3' -> [0, 1, 3] (the sysfs node-list format)."""
    out = []
    for part in text.strip().split(","):
        if not part:
            continue
        lo, _, hi = part.partition("-")
        out.extend(range(int(lo), int(hi or lo) + 1))
    return out


def memory_nodes() -> list:
    try:
        with open("/sys/devices/system/node/has_memory") as f:
            return parse_node_list(f.read())
    except OSError:
        return []


MPOL_INTERLEAVE = 3
_SYS_MBIND = {"x86_64": 237, "aarch64": 235}


def interleave_pages(address: int, nbytes: int, nodes: Optional[list] = None) -> bool:
    """Spread the (not yet touched) pages of a shared segment round-robin over the host's
    memory nodes (mbind MPOL_INTERLEAVE): every GPU of the node streams experts from it, so no
    single socket's DRAM serves all of them.  No-op (False) on a one-node host."""
    import ctypes
    import platform

    nodes = memory_nodes() if nodes is None else nodes
    nr = _SYS_MBIND.get(platform.machine())
    if len(nodes) < 2 or nr is None or nbytes <= 0:
        return False
    maxnode = max(nodes) + 1
    words = (maxnode + 63) // 64
    mask = (ctypes.c_ulong * words)()
    for n in nodes:
        mask[n // 64] |= 1 << (n % 64)
    libc = ctypes.CDLL(None, use_errno=True)
    libc.syscall.restype = ctypes.c_long
    rc = libc.syscall(ctypes.c_long(nr), ctypes.c_void_p(address), ctypes.c_ulong(nbytes),
                      ctypes.c_int(MPOL_INTERLEAVE), mask, ctypes.c_ulong(maxnode + 1),
                      ctypes.c_uint(0))
    return rc == 0


def open_shared_store(name: str, nbytes: int, local_rank: int,
                      barrier: Callable[[], None],
                      fill: Optional[Callable[[SharedExpertStore], None]] = None):
    """Local rank 0 creates (and fills) the segment; the others attach after a barrier.

    Returns the store; `fill(store)` runs on the owner before the barrier releases the rest.
    """
    if local_rank == 0:
        store = SharedExpertStore.create(name, nbytes)
        interleave_pages(store.address, store.nbytes)
        if fill is not None:
            fill(store)
        barrier()
        return store
    barrier()
    return SharedExpertStore.attach(name)


def open_shared_coded(name: str, engine, local_rank: int, barrier: Callable[[], None]):
    """The exponent-coded copy of a node-shared store: local rank 0 sizes, creates and encodes
    it through its engine; the other ranks attach after the barrier.  Returns the segment."""
    if local_rank == 0:
        seg = SharedExpertStore.create(name, engine.coded_size())
        interleave_pages(seg.address, seg.nbytes)
        engine.attach_coded(seg, build=True)
        barrier()
        return seg
    barrier()
    seg = SharedExpertStore.attach(name)
    engine.attach_coded(seg, build=False)
    return seg


def local_world() -> tuple:
    """(local_rank, local_world_size) from the torch.distributed.run environment."""
    return int(os.environ.get("LOCAL_RANK", "0")), int(os.environ.get("LOCAL_WORLD_SIZE", "1"))


def reduce_timing(elapsed_ms: float, tokens: int, world: int):
    """Whole-job throughput of independent replicas: all tokens / slowest rank's time."""
    if world == 1:
        return tokens / (elapsed_ms / 1e3), elapsed_ms, tokens
    import torch
    import torch.distributed as dist

    dev = "cuda" if (torch.cuda.is_available() and dist.get_backend() == "nccl") else "cpu"
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    n = torch.tensor([float(tokens)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    ms, total = float(t.item()), int(n.item())
    return total / (ms / 1e3), ms, total


def peer_home(layer: int, expert: int, num_experts: int, world: int) -> int:
    """The replica whose HBM holds the home copy of (layer, expert) in the peer tier: round robin
    over the node's ranks, so each GPU holds 1/world of the raw experts (8x7B on 8 GPUs: 11.3 GB)."""
    return (layer * num_experts + expert) % world


def open_peer_tier(engine, rank: int, world: int, all_gather_object: Callable, include_own: bool = False):
    """NVLink peer-HBM miss tier: every replica copies its home share of the raw
    experts from its host store into its own HBM once, publishes the buffer as a CUDA IPC handle,
    and maps the other replicas' buffers; the engine then serves misses of experts homed on a
    peer with device-to-device copies over NVLink instead of PCIe (moe_engine_attach_peer_tier).
    include_own also serves the rank's own home experts from its HBM (the one-GPU stand-in).
    all_gather_object(obj) -> [obj of rank 0, ..., rank world-1].  Returns (home tensor, blocks):
    keep both alive while the tier is attached."""
    import torch
    from torch.multiprocessing.reductions import reduce_tensor

    cfg = engine.config
    L, E = cfg.num_layers, cfg.num_experts
    mine = [(l, e) for l in range(L) for e in range(E) if peer_home(l, e, E, world) == rank]
    home = torch.empty((max(1, len(mine)), cfg.expert_bytes), dtype=torch.uint8, device=engine._dev)
    for i, (l, e) in enumerate(mine):
        home[i].copy_(torch.from_numpy(engine.expert_block(l, e)))
    torch.cuda.synchronize(engine._dev)
    handles = all_gather_object(reduce_tensor(home) if world > 1 else None)
    blocks = {}
    for r in range(world):
        if r == rank and not include_own:
            continue
        t = home if r == rank else handles[r][0](*handles[r][1])
        owned = [(l, e) for l in range(L) for e in range(E) if peer_home(l, e, E, world) == r]
        for i, le in enumerate(owned):
            blocks[le] = t[i]
    engine.attach_peer_tier(blocks)
    return home, blocks
