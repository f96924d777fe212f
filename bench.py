#!/usr/bin/env python
"""bench.py -- throughput of the B200 decimal -> binary64 parser (arXiv 2101.11408).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2] [--variant split|batch]

A step is one pass of the whole hot path over one
batch of synthetic input: parse_f64_split (record splitter + scanner +
Algorithm 1 + bracket + exact slow path) over config 2 -- 10^8 uniform [0,1)
binary64 values printed %.17g, newline separated (2.0 GB of text), the
configuration BASELINE.json's metric is quoted on.  Inputs are resident in HBM
when the timed region starts; they are larger than L2 (126 MB), so no flush is
needed between steps.  Rank 0 prints ONE JSON line.

N > 1 (torchrun, one process per GPU): weak scaling, every rank parses its own
independently seeded config-2 buffer; no data-path collective (records are
independent); the step time is the max over ranks.

--impl reference: the CPU oracle (oracle/, exact big-integer parser) on this
box's host cores, on bounded samples of the same workload (the paper has no
reference implementation to install).
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input GB/s and Gfloats/s parsed (bit-exact vs oracle); % of B200 HBM roofline"
WORKLOAD_DESC = {
    1: "config1: 1e5 uniform [0,1) binary64 printed %.17g, newline separated",
    2: "config2: 1e8 uniform [0,1) binary64 printed %.17g, newline separated (~2.0 GB)",
    3: "config3: 5e7 lon/lat fixed notation, 6-16 significant digits, comma/newline separated",
    4: "config4: 1e8 random-bit binary64 printed %.17e (+0.1% inf/nan)",
    5: "config5: 1e7 adversarial long strings (ties, tie+-1, 20-40 random digits)",
    6: "config6 (paper's 'integer' dataset, SURVEY 8f f2): 1e8 random 32-bit unsigned integers, newline separated",
    7: "config7 (paper's 'many digits' dataset, SURVEY 8f f2): 1e7 records of three random 64-bit integers in sequence",
    8: "config8 (SURVEY 8f f4): config 2's 1e8 uniform [0,1) values as C99 hex floats, newline separated",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--variant", choices=["split", "batch"], default="split")
    ap.add_argument("--grammar", choices=["default", "hex", "json"], default=None,
                    help="grammar option (*_ex calls); default: hex for config 8, else the default grammar")
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64",
                    help="output format: binary64 (headline) or binary32 (parse_f32_*, SURVEY 8(f) f1)")
    ap.add_argument("--n", type=int, default=None, help="override record count")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunk-mb", type=int, default=64, help="chunk size of the streaming host call")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--profile-run", action="store_true", help="few steps, no e2e / cpu (for ncu)")
    ap.add_argument("--shard", action="store_true",
                    help="N > 1: strong scaling -- ONE config stream cut at record starts across the ranks "
                         "(shard.py), each step parses the rank's shard and exchanges the record counts "
                         "(NCCL all_gather of one int64 per rank: the global output positions)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_entry(cfg, variant):
    """The committed ncu summary of the dominant kernel for this workload (binary64, default grammar)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get("config%d_%s" % (cfg, variant))
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index, period=0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr is not None:
            self._thr.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0, "source": "nvml unavailable"}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}


# --------------------------------------------------------------------------
def cpu_baseline(w, seconds, sep_mask):
    """The oracle, as it stands, on host cores over a bounded prefix of the workload."""
    import multiprocessing as mp
    import numpy as np
    from oracle.api import parse_split_pool
    procs = os.cpu_count() or 1
    raw = w.data

    def prefix(nbytes):
        end = min(int(nbytes), raw.size)
        while end < raw.size and raw[end - 1] != 10:
            end += 1
        return bytes(raw[:end])

    with mp.get_context("fork").Pool(procs) as pool:
        # probe the rate on ~8 MB, then time one pass over a prefix sized for `seconds`
        probe = prefix(8_000_000)
        t0 = time.perf_counter()
        parse_split_pool(probe, sep_mask, pool, procs * 4)
        rate = len(probe) / max(time.perf_counter() - t0, 1e-3)
        sample = prefix(rate * seconds)
        t0 = time.perf_counter()
        bits, st = parse_split_pool(sample, sep_mask, pool, procs * 8)
        dt = time.perf_counter() - t0
    nrec = bits.size
    ok = bool(np.array_equal(bits, w.exp_bits[:nrec])) if w.known[:nrec].all() else None
    # one core, on a 10^6-record sample (SURVEY.md 8(d) "Oracle timing")
    from oracle.api import _split_chunk
    one = prefix(min(raw.size, len(sample) * 1_000_000 // max(nrec, 1)))
    t1 = time.perf_counter()
    b1, _s1 = _split_chunk((one, sep_mask))
    dt1 = time.perf_counter() - t1
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"value": len(sample) / dt / 1e9, "unit": "GB/s", "cores": procs, "kind": "oracle",
            "cpu_model": model,
            "single_core": {"records": int(b1.size), "records_per_s": b1.size / dt1, "gb_per_s": len(one) / dt1 / 1e9,
                            "seconds": dt1},
            "sample": "first %d records (%.1f MB) of the same workload, one pass, %d processes"
                      % (nrec, len(sample) / 1e6, procs),
            "gfloats_per_s": nrec / dt / 1e9, "seconds": dt, "round_trip_ok": ok}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp
    import workloads
    from oracle.api import parse_split_pool
    procs = os.cpu_count() or 1
    n = min(args.n or workloads.CONFIG_N[args.config], 3_000_000)
    w = workloads.generate(args.config, n)
    data = bytes(w.data)
    # size a step to ~3 s of oracle work on this box
    with mp.get_context("fork").Pool(procs) as pool:
        probe = data[: min(len(data), 2_000_000)]
        while probe and probe[-1] != 10:
            probe = probe[:-1]
        t0 = time.perf_counter()
        parse_split_pool(probe, w.sep_mask, pool, procs * 4)
        rate = len(probe) / (time.perf_counter() - t0)
        step_bytes = int(min(len(data), max(1_000_000, rate * 3.0)))
        sample = data[:step_bytes]
        while sample and sample[-1] != 10:
            sample = sample[:-1]
        times, nrec = [], 0
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            bits, _st = parse_split_pool(sample, w.sep_mask, pool, procs * 4)
            dt = time.perf_counter() - t0
            nrec = bits.size
            if i >= args.warmup:
                times.append(dt)
    t = statistics.mean(times)
    val = len(sample) / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "python-int (exact rational)", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[args.config], "variant": "oracle split (CPU)",
                   "records_per_step": nrec, "text_bytes_per_step": len(sample)},
        "gfloats_per_s": nrec / t / 1e9,
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": procs, "kind": "oracle",
                         "sample": "first %d records (%.1f MB) of the workload per step" % (nrec, len(sample) / 1e6)},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import workloads
    from paper_2101_11408_b200 import native

    ws_n, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws_n > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    native.load()
    cfg = args.config
    n = args.n or workloads.CONFIG_N[cfg]
    shard_mode = args.shard and args.variant == "split"
    seed = cfg if (rank == 0 or shard_mode) else cfg + 1000 * rank
    t0 = time.perf_counter()
    w = workloads.generate(cfg, n, seed=seed)
    gen_s = time.perf_counter() - t0
    shard_info = None
    if shard_mode:  # this rank's byte range of the one stream (paper_2101_11408_b200/shard.py)
        from paper_2101_11408_b200 import shard
        a, b = shard.shard_range(w.data, ws_n, rank, w.sep_mask)
        i0, i1 = (int(x) for x in np.searchsorted(w.offsets, [a, b]))
        w = workloads.Workload(cfg, w.data[a:b], w.offsets[i0:i1] - a, w.sep_mask, w.exp_bits[i0:i1],
                               w.exp_status[i0:i1], w.known[i0:i1])
        n = i1 - i0
        shard_info = {"bytes": [a, b], "first_record": i0}
    L = int(w.data.size)
    host = torch.from_numpy(w.data).pin_memory()
    dev = host.to("cuda")
    dev_off = torch.from_numpy(w.offsets).to("cuda") if args.variant == "batch" else None
    f32 = args.dtype == "f32"
    ob = 4 if f32 else 8  # output bytes per record
    out = torch.empty(n, dtype=torch.float32 if f32 else torch.float64, device="cuda")
    status = torch.empty(n, dtype=torch.uint8, device="cuda")
    n_out = torch.zeros(1, dtype=torch.int64, device="cuda")
    if args.variant == "split":
        wsp = native.Workspace.for_split(L)
    else:
        wsp = native.Workspace.for_batch(L, n)
    stream = torch.cuda.current_stream()
    split_fn = native.parse_f32_split if f32 else native.parse_f64_split
    batch_fn = native.parse_f32_batch if f32 else native.parse_f64_batch
    gname = args.grammar or ("hex" if cfg == 8 else "default")
    grammar = {"default": 0, "hex": native.GRAMMAR_HEX, "json": native.GRAMMAR_JSON}[gname]

    counts = torch.zeros(ws_n, dtype=torch.int64, device="cuda")

    def step(stats=None):
        if args.variant == "split":
            split_fn(dev, w.sep_mask, capacity=n, out=out, status=status, n_out=n_out, ws=wsp, stats=stats,
                     stream=stream, grammar=grammar)
            if shard_mode and dist is not None:  # the only exchange: every rank's record count
                dist.all_gather_into_tensor(counts, n_out)
        else:
            batch_fn(dev, dev_off, out=out, status=status, ws=wsp, stats=stats, stream=stream, grammar=grammar)

    # correctness (untimed) on the instantiation the timed steps launch
    # (no stats), then the path counters in a separate run
    step()
    torch.cuda.synchronize()
    nrec = int(n_out.item()) if args.variant == "split" else n
    if not f32:
        got = out.view(torch.int64)
        known = torch.from_numpy(w.known.astype(np.bool_)).to("cuda")
        want = torch.from_numpy(w.exp_bits.view(np.int64)).to("cuda")
        mism = int(((got != want) & known).sum().item())
        mism_st = int(((status != torch.from_numpy(w.exp_status).to("cuda")) & known).sum().item())
        parity = {"records": nrec, "checked_by_construction": int(known.sum().item()),
                  "mismatches": mism + mism_st,
                  "against": "generator's source doubles (17-digit round trip, PAPER.md L55)"}
    else:
        # binary32: the oracle (exact decimal -> binary32) on an evenly spaced sample of records
        import oracle
        idx = np.unique(np.linspace(0, n - 1, num=min(n, 20000)).astype(np.int64))
        got = out.view(torch.int32).cpu().numpy().view(np.uint32)[idx]
        gst = status.cpu().numpy()[idx]
        offs = w.offsets
        raw = w.data
        mism = 0
        for k, i in enumerate(idx):
            e = int(offs[i + 1]) - 1 if i + 1 < n else int(raw.size) - (1 if raw[-1] == 10 else 0)
            bits, st = oracle.parse_record(bytes(raw[int(offs[i]):e]), "f32", grammar)
            mism += int(bits != int(got[k]) or st != int(gst[k]))
        parity = {"records": nrec, "checked_by_oracle": int(idx.size), "mismatches": mism,
                  "against": "oracle/ round_decimal32 on an evenly spaced sample of records"}
    stats = torch.zeros(native.NSTATS, dtype=torch.int64, device="cuda")
    step(stats)
    torch.cuda.synchronize()
    stat_vals = dict(zip(native.STAT_NAMES, [int(x) for x in stats.cpu().tolist()]))

    for _ in range(args.warmup):
        step()
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for e4 in ev:  # torch creates the CUDA events lazily: record once so the handles exist
        for e in e4:
            e.record(stream)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(K):
            ev[i][0].record(stream)
            native.set_profile_events(ev[i][1], ev[i][2], None)
            step()
            ev[i][3].record(stream)
        torch.cuda.synchronize()
    native.set_profile_events(None, None, None)
    if dist is not None:
        dist.barrier()
    total_ms = ev[0][0].elapsed_time(ev[K - 1][3])
    step_ms = [e[0].elapsed_time(e[3]) for e in ev]
    kern_ms = [e[1].elapsed_time(e[2]) for e in ev]
    ms = total_ms / K
    kms = statistics.mean(kern_ms)
    if dist is not None:
        t = torch.tensor([ms, kms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
        tot = torch.tensor([float(L), float(nrec)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tot)
        tot_bytes, tot_rec = float(tot[0]), float(tot[1])
    else:
        tot_bytes, tot_rec = float(L), float(nrec)

    # end to end through the C ABI with host buffers: H2D text, parse, D2H results.
    # split: the library's streaming host call (parse_*_split_host: chunked,
    # copies in both directions overlapping the parse), timed on the wall clock
    # around the whole synchronous call; batch: copy, parse, copy on the stream.
    e2e = None
    if not args.profile_run and args.e2e_steps > 0:
        out_h = torch.empty(n, dtype=out.dtype).pin_memory()
        st_h = torch.empty(n, dtype=torch.uint8).pin_memory()
        KE = args.e2e_steps
        host_fn = native.parse_f32_split_host if f32 else native.parse_f64_split_host
        if args.variant == "split":
            chunk = args.e2e_chunk_mb << 20
            host_fn(host, w.sep_mask, capacity=n, out=out_h, status=st_h, grammar=grammar, chunk_bytes=chunk,
                    stream=stream)  # warm-up (allocates the device slots once)
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(KE):
                _, _, _, nh = host_fn(host, w.sep_mask, capacity=n, out=out_h, status=st_h, grammar=grammar,
                                      chunk_bytes=chunk, stream=stream)
            ems = (time.perf_counter() - t0) * 1e3 / KE
            assert nh == nrec
            path = "pinned host text -> parse_%s_split_host (%d MiB chunks: H2D / k_split+k_slow / D2H " \
                   "overlapped) -> pinned host out/status" % (args.dtype, args.e2e_chunk_mb)
        else:
            nout_h = torch.empty(1, dtype=torch.int64).pin_memory()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for i in range(KE + 1):
                if i == 1:
                    if dist is not None:
                        dist.barrier()
                    torch.cuda.synchronize()
                    e0.record(stream)
                dev.copy_(host, non_blocking=True)
                step()
                out_h.copy_(out, non_blocking=True)
                st_h.copy_(status, non_blocking=True)
                nout_h.copy_(n_out, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            ems = e0.elapsed_time(e1) / KE
            path = "pinned host text -> cudaMemcpyAsync -> parse_%s_batch -> pinned host out/status" % args.dtype
        if dist is not None:
            t = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t[0])
        assert torch.equal(out_h[:64].view(torch.uint8), out[:64].cpu().view(torch.uint8))
        e2e = {"value": tot_bytes / (ems * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ems,
               "h2d_bytes_per_step": L, "d2h_bytes_per_step": (ob + 1) * n + (0 if args.variant == "split" else 8),
               "path": path}

    # latency: config 1 (1e5 records, 2 MB: L2-resident) through the same call,
    # median of 200 back-to-back calls timed with CUDA events
    lat = None
    if not args.profile_run and args.variant == "split" and not f32 and gname == "default":
        w1 = workloads.generate(1, seed=1)
        d1 = torch.from_numpy(w1.data).cuda()
        o1 = torch.empty(w1.n, dtype=torch.float64, device="cuda")
        s1 = torch.empty(w1.n, dtype=torch.uint8, device="cuda")
        n1 = torch.zeros(1, dtype=torch.int64, device="cuda")
        ws1 = native.Workspace.for_split(int(w1.data.size))
        for _ in range(10):
            native.parse_f64_split(d1, 1, capacity=w1.n, out=o1, status=s1, n_out=n1, ws=ws1, stream=stream)
        times = []
        for _ in range(200):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            native.parse_f64_split(d1, 1, capacity=w1.n, out=o1, status=s1, n_out=n1, ws=ws1, stream=stream)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3)
        ok1 = bool(np.array_equal(o1.cpu().numpy().view(np.uint64), w1.exp_bits))
        lat = {"config": WORKLOAD_DESC[1], "us_per_call_median": statistics.median(times),
               "us_per_call_min": min(times), "calls": len(times), "bit_exact": ok1,
               "gfloats_per_s": w1.n / (statistics.median(times) * 1e-6) / 1e9}
    peak, peak_src = measured_peak()
    alg_bytes = L + (ob + 1) * nrec + (8 * n if args.variant == "batch" else 0)
    achieved = alg_bytes / (kms * 1e-3) / 1e9
    ncu = ncu_entry(cfg, args.variant) if (not f32 and gname == "default") else None
    traffic = None if ncu is None else ncu.get("dram_bytes_per_launch")
    issue = None if ncu is None else ncu.get("smsp__issue_active.avg.pct_of_peak_sustained_active")
    line = {
        "metric": METRIC,
        "value": tot_bytes / (ms * 1e-3) / 1e9,
        "unit": "GB/s",
        "gfloats_per_s": tot_rec / (ms * 1e-3) / 1e9,
        "hbm_frac_step": (alg_bytes * (tot_bytes / L)) / (ms * 1e-3) / 1e9 / (peak * ws_n),
        "n_gpus": ws_n,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "ms_per_step_min": min(step_ms),
        "ms_per_step_median": statistics.median(step_ms),
        "higher_is_better": True,
        "scaling": "strong" if shard_mode else "weak",
        "vs_baseline": None,
        "dtype": "u64 (integer path; bytes -> binary32 bits)" if f32 else "u64 (integer path; bytes -> binary64 bits)",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[cfg],
                   "variant": "parse_%s_%s%s" % (args.dtype, args.variant, "" if gname == "default" else
                                                 "_ex (grammar %s)" % gname),
                   "records_per_gpu": nrec, "text_bytes_per_gpu": L,
                   "l2": "inputs larger than L2 (126 MB); no flush between steps",
                   "parallelism": ("one stream sharded at record starts, count all_gather (NCCL)" if shard_mode
                                   else "replicas: one independent buffer per GPU") if ws_n > 1 else "1 GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_split" if args.variant == "split" else "k_batch",
                     "kernel_ms": kms, "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_definition": "text + %d B out + 1 B status per record" % ob +
                                         (" + 8 B offsets" if args.variant == "batch" else ""),
                     "peak_source": peak_src,
                     "limiter": None if issue is None else
                     "instruction issue: %.0f%% issue-active under ncu (profiles/ncu_summary.json)" % issue},
        "gpu_launches": 2 * K,
        "clocks": clk.summary(),
        "parity": parity,
        "path_stats": stat_vals,
        "gen_seconds": gen_s,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if lat is not None:
        line["latency_c1"] = lat
    if shard_info is not None:
        cs = counts.cpu().tolist()
        shard_info["counts"] = cs
        shard_info["exclusive_prefix_ok"] = (sum(cs[:rank]) == shard_info["first_record"]) if dist is not None else True
        line["shard"] = shard_info
    if rank == 0 and ws_n == 1 and not args.no_cpu_baseline and not args.profile_run:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds, w.sep_mask)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.profile_run:
        args.steps, args.warmup = min(args.steps, 3), min(args.warmup, 1)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
