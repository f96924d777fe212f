"""Small end-to-end run of every entry point for compute-sanitizer (memcheck,
racecheck, synccheck): split / batch, binary64 / binary32, hex and JSON
grammars, unaligned buffers whose first record goes to the slow kernel,
long records across tiles, capacity cuts.  Checks results against the oracle
so a sanitizer-clean run is also a correct one."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2101_11408_b200 import native  # noqa: E402


def check(data, sep, fmt="f64", grammar=0, shift=0, capacity=None):
    raw = np.concatenate([np.zeros(shift, np.uint8), np.frombuffer(data, np.uint8)])
    dev = torch.from_numpy(raw).cuda()[shift:]
    fn = native.parse_f64_split if fmt == "f64" else native.parse_f32_split
    out, st, offs, n_out = fn(dev, sep, capacity=capacity, want_offsets=True, grammar=grammar)
    torch.cuda.synchronize()
    n = int(n_out.item())
    wo, res = oracle.parse_split(data, sep, fmt=fmt, grammar=grammar)
    assert n == len(wo), (n, len(wo))
    m = min(n, out.numel())
    u = np.uint64 if fmt == "f64" else np.uint32
    got = out[:m].cpu().numpy().view(u)
    assert np.array_equal(got, np.array([r[0] for r in res[:m]], dtype=u)), "split bits"
    assert np.array_equal(st[:m].cpu().numpy(), np.array([r[1] for r in res[:m]], dtype=np.uint8)), "split status"
    bf = native.parse_f64_batch if fmt == "f64" else native.parse_f32_batch
    o = torch.tensor(wo, dtype=torch.int64, device="cuda")
    out2, st2 = bf(dev, o, grammar=grammar)
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy().view(u), np.array([r[0] for r in res], dtype=u)), "batch bits"
    return n


def main():
    torch.cuda.set_device(0)
    native.load()
    total = 0
    for cfg, n in ((1, 3000), (3, 3000), (4, 3000), (5, 400), (6, 3000), (7, 500)):
        d = bytes(workloads.generate(cfg, n).data)
        for shift in (0, 7):
            total += check(d, workloads.CONFIG_SEP_MASK[cfg], shift=shift)
        total += check(d, workloads.CONFIG_SEP_MASK[cfg], fmt="f32")
    total += check(bytes(workloads.generate(8, 3000).data), 1, grammar=native.GRAMMAR_HEX)
    total += check(bytes(workloads.generate(4, 3000).data), 1, grammar=native.GRAMMAR_JSON)
    first = b"1." + b"3" * 90 + b"e-5\n" + b"12345678901234567890123e-300\n"
    for shift in (1, 9, 15):
        total += check(first + bytes(workloads.generate(5, 200).data), 1, shift=shift)
    longs = b"\n".join([b"0." + b"0" * 6000 + b"1e6001", b"7" * 9000, b"1e" + b"0" * 5000 + b"5", b"-inf", b""])
    total += check(longs + b"\n" + bytes(workloads.generate(2, 2000).data), 1)
    total += check(bytes(workloads.generate(5, 400).data), 1, capacity=123)
    dense = b"".join(b"%d\n" % (i % 10) for i in range(20000))
    total += check(dense, 1)
    print("sanitize run ok: %d records" % total)


if __name__ == "__main__":
    main()
