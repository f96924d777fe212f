"""Helpers for the GPU parity tests: run the CUDA path, run the oracle, compare."""
import numpy as np
import torch

import oracle


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


_UINT = {"f64": np.uint64, "f32": np.uint32}


def gpu_batch(data, offsets, stats=None, fmt="f64", grammar=0):
    from paper_2101_11408_b200 import native
    d = to_dev(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data)
    o = to_dev(np.asarray(offsets, dtype=np.int64))
    ws = native.Workspace.for_batch(d.numel(), o.numel()) if stats is not None else None
    fn = native.parse_f64_batch if fmt == "f64" else native.parse_f32_batch
    out, st = fn(d, o, ws=ws, stats=stats, grammar=grammar)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(_UINT[fmt]), st.cpu().numpy()


def gpu_split(data, sep_mask, stats=None, want_offsets=True, capacity=None, fmt="f64", grammar=0):
    from paper_2101_11408_b200 import native
    d = to_dev(np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data)
    ws = native.Workspace.for_split(d.numel()) if stats is not None else None
    fn = native.parse_f64_split if fmt == "f64" else native.parse_f32_split
    out, st, offs, n_out = fn(d, sep_mask, capacity=capacity, ws=ws, stats=stats, want_offsets=want_offsets,
                              grammar=grammar)
    torch.cuda.synchronize()
    n = int(n_out.item())
    m = min(n, out.numel())
    return (n, out[:m].cpu().numpy().view(_UINT[fmt]), st[:m].cpu().numpy(),
            None if offs is None else offs[:m].cpu().numpy())


def oracle_batch(data, offsets, procs=8, fmt="f64", grammar=0):
    res = oracle.parse_batch(bytes(data), list(map(int, offsets)), procs=procs, fmt=fmt, grammar=grammar)
    return (np.array([r[0] for r in res], dtype=_UINT[fmt]), np.array([r[1] for r in res], dtype=np.uint8))


def oracle_split(data, sep_mask, procs=8, fmt="f64", grammar=0):
    offs, res = oracle.parse_split(bytes(data), sep_mask, procs=procs, fmt=fmt, grammar=grammar)
    return (np.array(offs, dtype=np.int64), np.array([r[0] for r in res], dtype=_UINT[fmt]),
            np.array([r[1] for r in res], dtype=np.uint8))


def assert_same(got_bits, got_st, want_bits, want_st, data=None, offsets=None, what=""):
    assert got_bits.shape == want_bits.shape, (what, got_bits.shape, want_bits.shape)
    bad = np.nonzero((got_bits != want_bits) | (got_st != want_st))[0]
    if bad.size:
        lines = []
        for i in bad[:8]:
            rec = ""
            if data is not None and offsets is not None:
                s = int(offsets[i])
                e = int(offsets[i + 1]) if i + 1 < len(offsets) else len(data)
                rec = bytes(data[s:min(e, s + 80)])
            lines.append("  #%d %r got %016x/%d want %016x/%d" % (
                i, rec, int(got_bits[i]), int(got_st[i]), int(want_bits[i]), int(want_st[i])))
        raise AssertionError("%s: %d mismatches of %d\n%s" % (what, bad.size, got_bits.size, "\n".join(lines)))
