"""Multi-process (gloo, world_size 2, CPU) coverage of the replica plumbing bench.py uses on
N GPUs: disjoint request streams, the max-over-ranks / sum-of-tokens reduction, and the
node-shared expert store (local rank 0 creates and fills, the other ranks attach)."""
import os
import platform
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_05814_b200 import replicas
from paper_2511_05814_b200.engine import EngineConfig


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # shared store: rank 0 writes a pattern, rank 1 must see it after the barrier
        def fill(store):
            np.frombuffer(store.shm.buf, dtype=np.uint8)[:] = np.arange(store.nbytes) % 251

        store = replicas.open_shared_store(name, 1 << 20, rank, dist.barrier, fill)
        view = np.frombuffer(store.shm.buf, dtype=np.uint8)
        ok = bool(np.array_equal(view, np.arange(1 << 20) % 251))
        del view
        dist.barrier()
        store.close()
        # timing reduction: rank r took (r+1)*100 ms for (r+1)*8 tokens
        tps, ms, total = replicas.reduce_timing((rank + 1) * 100.0, (rank + 1) * 8, world)
        out[rank] = (ok, tps, ms, total, replicas.rank_token_base(rank))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_replicas():
    world = 2
    port = _free_port()
    name = "moeb200_test_%d" % os.getpid()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, name, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        ok, tps, ms, total, base = res[rank]
        assert ok, "attached replica does not see the owner's store contents"
        assert ms == 200.0 and total == 24
        assert tps == pytest.approx(24 / 0.2)
    assert res[0][4] != res[1][4]
    assert abs(res[1][4] - res[0][4]) >= replicas.TOKENS_PER_RANK_STREAM


def test_store_name_is_shape_specific():
    a = EngineConfig.mixtral_8x7b()
    b = EngineConfig.mixtral_8x22b()
    assert replicas.store_name(a, 42) != replicas.store_name(b, 42)
    assert replicas.store_name(a, 42) != replicas.store_name(a, 43)
    assert replicas.store_name(a, 42) == replicas.store_name(a, 42)
    assert replicas.store_name(a, 42).startswith("moeb200_")


def test_store_create_replaces_stale_segment():
    name = "moeb200_stale_%d" % os.getpid()
    s1 = replicas.SharedExpertStore.create(name, 4096)
    s1.shm.buf[0] = 7
    s1.shm.close()           # "killed" run: never unlinked
    s2 = replicas.SharedExpertStore.create(name, 8192)
    assert s2.nbytes >= 8192 and s2.shm.buf[0] == 0
    s2.close()


def test_node_list_parsing():
    assert replicas.parse_node_list("0") == [0]
    assert replicas.parse_node_list("0-1,3\n") == [0, 1, 3]
    assert replicas.parse_node_list("") == []


def test_interleave_pages_mbind():
    import mmap
    import ctypes

    m = mmap.mmap(-1, 1 << 21)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
    assert replicas.interleave_pages(addr, 1 << 21, nodes=[0]) is False   # one node: no-op
    if platform.machine() in ("x86_64", "aarch64"):
        # the syscall path itself (interleave over node 0 twice is valid on any host)
        assert replicas.interleave_pages(addr, 1 << 21, nodes=[0, 0]) is True
