"""Sharding one input across ranks (host logic).

Split variant (parse_f64_split): one byte stream cut into W ranges.

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


# ---------------------------------------------------------------------------
# Batch variant (parse_f64_batch; SURVEY.md 8(e) "offsets variant"): the record
# index range is split evenly; rank r parses records [i_r, i_{r+1}) and reads
# only bytes [offsets[i_r], end of record i_{r+1}-1).  No exchange is needed:
# the global index of the rank's first record is i_r.

def batch_shard(n, world, rank):
    """Record index range [i_r, i_{r+1}) of rank `rank`."""
    return n * rank // world, n * (rank + 1) // world


def batch_shard_bytes(offsets, length, i0, i1):
    """The byte range [lo, hi) and the rebased offsets rank shard [i0, i1) of a
    batch input parses.  Record i is [offsets[i], offsets[i+1]) (or
    [offsets[n-1], length)); out-of-range bounds make it INVALID.

    Every in-range bound of the shard's records lies in [lo, hi], so rebasing
    by lo keeps each record's bounds -- and validity -- exactly; out-of-range
    starts become -1 (still out of range).  When i1 < n the end of record
    i1-1 is offsets[i1], passed as one extra record start whose result the
    caller drops (`extra`)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    n = offsets.shape[0]
    if i0 >= i1:
        return 0, 0, np.zeros(0, dtype=np.int64), False
    extra = i1 < n
    bounds = offsets[i0:i1 + 1] if extra else offsets[i0:i1]
    inr = (bounds >= 0) & (bounds <= length)
    vals = bounds[inr]
    lo = int(vals.min()) if vals.size else 0
    hi = length if not extra else (int(vals.max()) if vals.size else lo)
    reb = np.where(inr, bounds - lo, -1).astype(np.int64)
    return lo, hi, reb, extra


def parse_sharded_batch(data, offsets, parse_fn, group=None):
    """Parse this rank's share of a batch input (offsets variant).

    parse_fn(bytes_u8, rebased_offsets) -> (bits, status) parses one shard (on a
    GPU: native.parse_f64_batch).  Returns (first_index, bits, status)."""
    import torch.distributed as dist
    n = len(offsets)
    i0, i1 = batch_shard(n, dist.get_world_size(group), dist.get_rank(group))
    if i1 <= i0:
        return i0, np.zeros(0, dtype=np.uint64), np.zeros(0, dtype=np.uint8)
    lo, hi, reb, extra = batch_shard_bytes(offsets, data.shape[0], i0, i1)
    bits, status = parse_fn(data[lo:hi], reb)
    if extra:
        bits, status = bits[:-1], status[:-1]
    return i0, np.asarray(bits), np.asarray(status)


def native_split_fn(device="cuda"):
    """parse_fn for parse_sharded running native.parse_f64_split on `device`."""
    from . import native

    def fn(buf, sep_mask):
        d = torch.from_numpy(np.ascontiguousarray(buf)).to(device)
        out, st, offs, n_out = native.parse_f64_split(d, sep_mask, want_offsets=True)
        n = int(n_out.item())
        return (out[:n].cpu().numpy().view(np.uint64), st[:n].cpu().numpy(), offs[:n].cpu().numpy())
    return fn

