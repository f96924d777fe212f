"""Multi-rank sharding of the split variant on CPU (gloo, world_size 2).

Host logic only: byte cuts moved to record starts,
per-rank parse, exclusive scan of record counts by all_gather.  The per-rank
parse here is the CPU oracle (test infrastructure); on GPUs it is
native.parse_f64_split.  The gathered result must equal the unsharded parse.
"""
import os
import random
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2101_11408_b200 import shard


def _oracle_parse(buf, sep_mask):
    offs, res = oracle.parse_split(bytes(buf), sep_mask)
    return (np.array([r[0] for r in res], dtype=np.uint64), np.array([r[1] for r in res], dtype=np.uint8),
            np.array(offs, dtype=np.int64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for data, mask in cases:
            arr = np.frombuffer(data, dtype=np.uint8)
            first, total, bits, st, starts = shard.parse_sharded(arr, mask, _oracle_parse)
            out.append((first, total, bits.tolist(), st.tolist(), starts.tolist()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _cases():
    rng = random.Random(7)
    cases = [(b"", 0), (b"\n", 1), (b"1\n", 1), (b"1\n2", 1), (b"\n\n\n,\n", 0), (b"1.5,2.5\n3.5", 0),
             (b"1.5,2.5\n3.5", 1), (b"12345678901234567890\n" * 3, 1)]
    parts = []
    for _ in range(400):
        parts.append(rng.choice([b"0.5", b"-1e3", b"inf", b"", b"x", b"3.14159", b"1" * rng.randint(1, 40)]))
        parts.append(rng.choice([b"\n", b",", b"\r\n"]))
    big = b"".join(parts)
    cases += [(big, 0), (big, 1), (big, 2), (big[:-1], 3)]
    return cases


@pytest.mark.parametrize("world", [2])
def test_sharded_split_matches_unsharded(world):
    cases = _cases()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (data, mask) in enumerate(cases):
        want_b, want_s, want_o = _oracle_parse(np.frombuffer(data, dtype=np.uint8), mask)
        got_b, got_s, got_o = [], [], []
        expect_first = 0
        for r in range(world):
            first, total, b, s, o = res[r][ci]
            assert first == expect_first and total == len(want_b), (ci, r)
            expect_first += len(b)
            got_b += b
            got_s += s
            got_o += o
        assert got_b == want_b.tolist() and got_s == want_s.tolist() and got_o == want_o.tolist(), ci


def test_record_boundary():
    d = np.frombuffer(b"ab\ncd,ef\n", dtype=np.uint8)
    assert shard.record_boundary(d, 0, 0) == 0
    assert shard.record_boundary(d, 1, 0) == 3
    assert shard.record_boundary(d, 3, 0) == 3
    assert shard.record_boundary(d, 4, 0) == 6
    assert shard.record_boundary(d, 4, 1) == 9
    assert shard.record_boundary(d, 9, 0) == 9


# ---------------------------------------------------------------------------
# offsets (batch) variant: records split evenly by index, no exchange
def _oracle_batch(buf, offs):
    res = oracle.parse_batch(bytes(buf), [int(o) for o in offs])
    return np.array([r[0] for r in res], dtype=np.uint64), np.array([r[1] for r in res], dtype=np.uint8)


def _batch_worker(rank, world, port, cases, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for data, offs in cases:
            arr = np.frombuffer(data, dtype=np.uint8)
            first, bits, st = shard.parse_sharded_batch(arr, offs, _oracle_batch)
            out.append((first, bits.tolist(), st.tolist()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _batch_cases():
    rng = random.Random(11)
    recs = [rng.choice([b"0.5\n", b"-1e3,", b"inf\n", b"\n", b"x", b"3.14159\r\n", b"1" * rng.randint(1, 40) + b"\n"])
            for _ in range(500)]
    data = b"".join(recs)
    offs, pos = [], 0
    for r in recs:
        offs.append(pos)
        pos += len(r)
    zig = list(offs)
    for i in rng.sample(range(len(zig)), 60):  # decreasing, negative, past-the-end bounds
        zig[i] = rng.choice([-5, len(data) + 3, zig[max(0, i - 3)], len(data), 0])
    return [(data, offs), (data, zig), (data, offs[:1]), (data, []), (b"", [0, 0])]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_batch_matches_unsharded(world):
    cases = _batch_cases()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (data, offs) in enumerate(cases):
        want_b, want_s = _oracle_batch(np.frombuffer(data, dtype=np.uint8), offs)
        got_b, got_s, expect_first = [], [], 0
        for r in range(world):
            first, b, s = res[r][ci]
            assert first == expect_first, (ci, r)
            expect_first += len(b)
            got_b += b
            got_s += s
        assert got_b == want_b.tolist() and got_s == want_s.tolist(), ci
