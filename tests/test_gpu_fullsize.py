"""Full-size bit-exact gate ("out bits and status bytes must
equal the oracle's for all n records in every config") in the launch
configuration bench.py times (parse_f64_split with a reusable workspace).

Every record is checked:
  * records whose answer is known by construction -- configs 2, 4 and 8 by the
    17-digit round trip / exact hex printing, config 6 (exact
    integers), config 5's ties and tie+-1 neighbours (PAPER.md L45-46
    generalised) -- against the construction;
  * every record of configs 3, 5 and 7 against the CPU oracle, run over the
    whole buffer on all host cores (oracle.api.parse_split_pool; about 15 s for
    config 3 on 16 cores);
and the split offsets must equal the generator's record starts.
"""
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

import workloads

pytestmark = pytest.mark.gpu


def _run_split(w, grammar=0):
    from paper_2101_11408_b200 import native
    dev = torch.from_numpy(w.data).cuda()
    n = w.n
    ws = native.Workspace.for_split(dev.numel())
    out, st, offs, n_out = native.parse_f64_split(dev, w.sep_mask, capacity=n, ws=ws, want_offsets=True,
                                                  grammar=grammar)
    torch.cuda.synchronize()
    res = (int(n_out.item()), out.cpu().numpy().view(np.uint64), st.cpu().numpy(), offs.cpu().numpy())
    del dev, out, st, offs, ws
    torch.cuda.empty_cache()
    return res


def _oracle_all(w):
    from oracle.api import parse_split_pool
    procs = os.cpu_count() or 1
    with mp.get_context("fork").Pool(procs) as pool:
        return parse_split_pool(bytes(w.data), w.sep_mask, pool, procs * 8)


def _first_bad(bits, st, wb, ws, mask=None):
    bad = (bits != wb) | (st != ws)
    if mask is not None:
        bad &= mask
    return np.nonzero(bad)[0]


@pytest.mark.parametrize("cfg", [2, 3, 4, 5, 6, 7, 8])
def test_fullsize_split(cuda_lib, cfg):
    w = workloads.generate(cfg)
    from paper_2101_11408_b200 import native
    grammar = native.GRAMMAR_HEX if cfg == 8 else 0
    n_out, bits, st, offs = _run_split(w, grammar)
    assert n_out == w.n
    assert np.array_equal(offs, w.offsets)
    k = w.known.astype(bool)
    bad = _first_bad(bits, st, w.exp_bits, w.exp_status, k)
    assert bad.size == 0, "config %d: %d constructed mismatches, first %s" % (cfg, bad.size, bad[:5])
    if k.all():
        return
    assert cfg in (3, 5, 7), cfg
    wb, ws = _oracle_all(w)
    assert wb.size == w.n
    bad = _first_bad(bits, st, wb, ws)
    ends = np.append(w.offsets[1:], w.data.size)
    msg = ["#%d %r got %016x/%d want %016x/%d" % (i, bytes(w.data[w.offsets[i]:min(ends[i], w.offsets[i] + 60)]),
                                                   int(bits[i]), int(st[i]), int(wb[i]), int(ws[i]))
           for i in bad[:5]]
    assert bad.size == 0, "config %d: %d of %d records differ from the oracle\n%s" % (cfg, bad.size, w.n,
                                                                                       "\n".join(msg))


def test_fullsize_batch_config4(cuda_lib):
    from paper_2101_11408_b200 import native
    w = workloads.generate(4)
    dev = torch.from_numpy(w.data).cuda()
    o = torch.from_numpy(w.offsets).cuda()
    out, st = native.parse_f64_batch(dev, o)
    torch.cuda.synchronize()
    bits = out.cpu().numpy().view(np.uint64)
    assert np.array_equal(bits, w.exp_bits) and np.array_equal(st.cpu().numpy(), w.exp_status)
