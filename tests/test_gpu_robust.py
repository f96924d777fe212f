"""GPU robustness and grammar-edge parity.

* G9 exponent saturation: 13-, 25-, 5000-digit exponents and the compensating
  form 0.<N zeros>1e<N+1> (N up to 10^5) must give the exact value (PAPER.md
  L179: the exponent is unbounded; the kernels clamp at bounds larger than any
  record, G9) -- through the common-case parser (records of at most
  64 bytes) and the slow kernel's lexer (longer records).
* Concurrency: two split calls on two streams with their own workspaces,
  in flight together (the look-back's forward progress, k_common.cuh).
* An unaligned buffer whose FIRST record goes to the slow kernel: its staging
  must not read before bytes[0] (compute-sanitizer run in
  profiles/).
* The Clinger ablation builds pass the
  oracle parity of test_configs_vs_oracle / test_random_w_q in a subprocess.
"""
import os
import random
import subprocess
import sys

import numpy as np
import pytest
import torch

import workloads
from tests.gpu_helpers import gpu_batch, gpu_split, oracle_batch, oracle_split, assert_same, to_dev

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _buffer(recs, sep=b"\n"):
    offs, pos, parts = [], 0, []
    for r in recs:
        offs.append(pos)
        parts.append(r + sep)
        pos += len(r) + len(sep)
    return b"".join(parts), np.array(offs, dtype=np.int64)


def _both(data, offs, sep_mask, what):
    gb, gs = gpu_batch(data, offs)
    wb, ws = oracle_batch(data, offs)
    assert_same(gb, gs, wb, ws, data, offs, what + " [batch]")
    n, sb, ss, so = gpu_split(data, sep_mask)
    wo, wb2, ws2 = oracle_split(data, sep_mask)
    assert n == len(wo) and np.array_equal(so, wo), what
    assert_same(sb, ss, wb2, ws2, data, wo, what + " [split]")


def _g9_records():
    recs = []
    for nd in (13, 25, 60, 5000):
        z = "0" * (nd - 1)
        nines = "9" * nd
        for mant in ("1", "2.5", "-7.25", "0.001", "123456789012345678", "1" + "0" * 70 + "3"):
            for ex in (z + "5", "-" + z + "5", "+" + z + "17", nines, "-" + nines, z + "0"):
                recs.append(("%se%s" % (mant, ex)).encode())
        recs.append(("0e" + nines).encode())
        recs.append(("-0.000E-" + nines).encode())
    for N in (10, 50, 300, 5000, 100_000):
        recs.append(("0." + "0" * N + "1e" + str(N + 1)).encode())
        recs.append(("1" + "0" * N + "e-" + str(N)).encode())
        recs.append(("0." + "0" * N + "15e" + str(N + 1)).encode())
        recs.append(("-0." + "0" * N + "2225073858507201e" + str(N - 307)).encode())
    return recs


def test_g9_exponent_saturation(cuda_lib):
    recs = _g9_records()
    assert any(len(r) <= 64 for r in recs) and any(len(r) > 64 for r in recs)
    data, offs = _buffer(recs)
    _both(data, offs, 1, "G9 exponents")
    # the same records between ordinary ones (the fast kernel's tiles, halos)
    rng = random.Random(9)
    mixed = []
    for r in recs:
        mixed += [("%.17g" % rng.random()).encode() for _ in range(rng.randrange(0, 300))]
        mixed.append(r)
    data, offs = _buffer(mixed)
    _both(data, offs, 1, "G9 exponents mixed")


def test_two_streams_concurrent(cuda_lib):
    # two large split calls in flight together on two streams (each with its
    # own workspace): results equal the stream-serial ones and the construction
    from paper_2101_11408_b200 import native
    wa = workloads.generate(2, 4_000_000, seed=21)
    wb = workloads.generate(4, 3_000_000, seed=22)
    da, db = to_dev(wa.data), to_dev(wb.data)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    wsa, wsb = native.Workspace.for_split(da.numel()), native.Workspace.for_split(db.numel())
    res = {}
    torch.cuda.synchronize()
    for rep in range(3):
        with torch.cuda.stream(sa):
            ra = native.parse_f64_split(da, 1, capacity=wa.n, ws=wsa, stream=sa)
        with torch.cuda.stream(sb):
            rb = native.parse_f64_split(db, 1, capacity=wb.n, ws=wsb, stream=sb)
        torch.cuda.synchronize()
        for name, r, w in (("a", ra, wa), ("b", rb, wb)):
            out, st, _, n_out = r
            assert int(n_out.item()) == w.n
            bits = out.cpu().numpy().view(np.uint64)
            assert np.array_equal(bits, w.exp_bits) and np.array_equal(st.cpu().numpy(), w.exp_status), (name, rep)
            res.setdefault(name, bits)


@pytest.mark.parametrize("shift", [1, 5, 9, 15])
def test_unaligned_first_record_slow(cuda_lib, shift):
    # the first record is long (> 64 bytes) or has more than 19 digits: the slow
    # kernel stages it from the 16-byte grid below bytes[0]
    from paper_2101_11408_b200 import native
    first = [b"1." + b"3" * 90 + b"e-5", b"12345678901234567890123e-300", b"0." + b"0" * 80 + b"7e81"]
    for f in first:
        body = f + b"\n" + bytes(workloads.generate(5, 2000).data)
        raw = np.concatenate([np.zeros(shift, np.uint8), np.frombuffer(body, np.uint8)])
        dev = to_dev(raw)[shift:]
        assert dev.data_ptr() % 16 == shift % 16
        data = raw[shift:]
        out, st, offs, n_out = native.parse_f64_split(dev, 1, want_offsets=True)
        torch.cuda.synchronize()
        n = int(n_out.item())
        wo, wb, ws = oracle_split(data, 1)
        assert n == len(wo)
        assert_same(out[:n].cpu().numpy().view(np.uint64), st[:n].cpu().numpy(), wb, ws, data, wo, "first slow")
        out2, st2 = native.parse_f64_batch(dev, to_dev(wo))
        torch.cuda.synchronize()
        assert_same(out2.cpu().numpy().view(np.uint64), st2.cpu().numpy(), wb, ws, data, wo, "first slow batch")


def _variant_lib(name, defines):
    from paper_2101_11408_b200 import build
    path = os.path.join(build.HERE, "libfpparse_%s.so" % name)
    newest = max(os.path.getmtime(f) for f in build.sources())
    if not os.path.exists(path) or os.path.getmtime(path) < newest:
        build.build_variant(name, defines)
    return path


@pytest.mark.parametrize("name,defines", [("clinger", ["FPP_CLINGER=1"]), ("clvote", ["FPP_CLINGER=2"])])
def test_clinger_variants_parity(cuda_lib, name, defines):
    # Clinger's fast path as a build variant;
    # the oracle parity suite runs against it in a fresh process (FPP_LIB)
    lib = _variant_lib(name, defines)
    env = dict(os.environ, FPP_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_gpu_parity.py::test_configs_vs_oracle",
                        "tests/test_gpu_parity.py::test_random_w_q",
                        "tests/test_gpu_f32.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_lookback_fallback_parity(cuda_lib):
    """The look-back's forward-progress fallback (k_common.cuh: a predecessor
    still unpublished after kSpinLimit polls is counted from global memory
    and published by CAS) never triggers in normal runs; a build with
    kSpinLimit = 1 takes it on every wait.  Its results must equal the
    oracle's and the construction."""
    lib = _variant_lib("lbfall", ["FPP_SPIN_LIMIT=1"])
    env = dict(os.environ, FPP_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_gpu_parity.py::test_configs_vs_oracle",
                        "tests/test_gpu_parity.py::test_separators_at_tile_edges",
                        "tests/test_gpu_parity.py::test_determinism_and_stats",
                        "tests/test_gpu_robust.py::test_two_streams_concurrent"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout

