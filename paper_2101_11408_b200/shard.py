"""Sharding one byte stream across ranks for parse_f64_split (host logic).

Records are independent, so the only exchange a sharded split needs is the
exclusive scan of the ranks' record counts (one int64 per rank, gathered with
torch.distributed; NCCL over NVLink on GPUs, gloo in the CPU tests).

Rank r owns the records that START in [cut_r, cut_{r+1}), cut_r = len*r//W.
A record starts at p when p == 0 or bytes[p-1] is a separator (DESIGN.md
"Record grammar"), so rank r parses the byte range [a_r, a_{r+1}) with
a_r = the first record start >= cut_r (or len): the last record of a rank
ends at the separator just before a_{r+1}, and a final trailing separator
creates no record, exactly as in the unsharded stream.
"""
import numpy as np
import torch


def sep_bytes(sep_mask):
    m = 3 if sep_mask == 0 else sep_mask
    return [b for b, bit in ((10, 1), (44, 2)) if m & bit]


def record_boundary(data, pos, sep_mask):
    """First record start >= pos (or len).  data: 1-D uint8 numpy array."""
    n = data.shape[0]
    if pos <= 0:
        return 0
    if pos >= n:
        return n
    seps = sep_bytes(sep_mask)
    window = 4096
    p = pos
    while p < n:
        chunk = data[p - 1:min(n, p - 1 + window)]
        hit = np.nonzero(np.isin(chunk, seps))[0]
        if hit.size:
            return min(n, p + int(hit[0]))
        p += window
    return n


def shard_range(data, world, rank, sep_mask):
    """Byte range [a_r, a_{r+1}) rank `rank` parses."""
    n = data.shape[0]
    a = record_boundary(data, n * rank // world, sep_mask)
    b = record_boundary(data, n * (rank + 1) // world, sep_mask) if rank + 1 < world else n
    return a, max(a, b)


def exclusive_prefix(count, group=None, device="cpu"):
    """(first global record index of this rank, total records) via all_gather."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    mine = torch.tensor([int(count)], dtype=torch.int64, device=device)
    allc = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    counts = [int(c.item()) for c in allc]
    r = dist.get_rank(group)
    return sum(counts[:r]), sum(counts)


def parse_sharded(data, sep_mask, parse_fn, group=None, device="cpu"):
    """Parse this rank's shard of the global stream `data` (uint8 numpy array).

    parse_fn(shard_bytes_u8, sep_mask) -> (bits uint64[k], status uint8[k],
    starts int64[k]) parses one byte range (on a GPU: native.parse_f64_split).
    Returns (first_index, total, bits, status, global_starts).
    """
    import torch.distributed as dist
    a, b = shard_range(data, dist.get_world_size(group), dist.get_rank(group), sep_mask)
    bits, status, starts = parse_fn(data[a:b], sep_mask)
    first, total = exclusive_prefix(len(bits), group, device)
    return first, total, bits, status, np.asarray(starts, dtype=np.int64) + a
