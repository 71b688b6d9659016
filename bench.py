#!/usr/bin/env python
"""bench.py -- full-decode throughput of the learned-compression decoder on B200.

One step = one lc_decode launch over the whole BASELINE config-4 list (N = 5e8 u64 keys, Zipf
clusters, eps = 31; the largest config): read the compressed blob once, write N keys once.
Metric (BASELINE.json): full-decode GB/s = (compressed bytes + N * 8) / t, plus keys/s and the
fraction of the measured HBM copy peak.  Beside the headline, `decode_configs` times configs 2
and 3 (the other 1e8+-key configs of the north-star target), `access` times config 5's random
access and range decodes (plus quantiles, successor search, intersection, union) and
`free_intercept` config 2 under FORMAT F7.

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--config 1..5]

Under torchrun (N > 1) the list is sharded (strong scaling): every rank uploads only its
1024-aligned span's slices of the blob (lc_shard_upload) and decodes them, with no collective
on the data path; the time is the max over ranks of the device-timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full-decode GB/s (+keys/s) and % of HBM peak; random-access lookups/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _ncu_traffic(cid):
    """dram bytes per launch of the decode kernel from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(f"config{cid}")
    except Exception:
        return None


class ClockSampler:
    """NVML sampler of SM clock + throttle reasons while the timed region runs."""

    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
        0x1: "gpu_idle",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def _spec(cid):
    from synth import CONFIGS
    s = CONFIGS[cid]
    return s


def _workload_name(cid):
    s = _spec(cid)
    return f"config{cid}: N={s.n:.0e} u{s.key_bits} keys, {s.desc}, eps={s.eps}"


def _config_dict(cid, n, blob_len, L, b, ws):
    """The line's `config` (identical for both arms: same workload, same blob bytes)."""
    spec = _spec(cid)
    w = spec.key_bits // 8
    alg = blob_len + n * w
    return {"workload": _workload_name(cid), "n": n, "key_bits": spec.key_bits, "eps": spec.eps,
            "res_bits": b, "segments": L, "blob_bytes": blob_len, "bits_per_int": 8 * blob_len / n,
            "ratio_r": blob_len / (n * w), "bytes_per_step": alg,
            "l2": ("no flush: every step reads+writes %.2f GB >> 126 MB L2" % (alg / 1e9))
            if alg > 4 * 126e6 else "L2 not flushed: the step's %.1f MB are not >> the 126 MB L2 "
            "(small informational config)" % (alg / 1e6),
            "parallelism": "single GPU" if ws == 1 else
            f"shards x{ws} (strong: each GPU holds and decodes 1/{ws} of the list)"}


def _kernel_name(h):
    """Symbol of the full-decode instantiation lc_decode picks for header h (lc_kernels.cu:
    dense / sparse by segment density, one instantiation per key width and residual width)."""
    k64 = int(h.key_bits == 64)
    sparse = int(h.n_seg * 64 < h.n)
    return f"lc_decode_kernel<{k64},{int(h.res_bits)},{sparse},0>"


def _env_dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle (plain C, OpenMP over 65536-key spans) timed on the host cores: the same
    metric, config and units as the GPU arm.  Rank 0 only."""
    ws, rank, _ = _env_dist()
    if rank != 0:
        return
    from oracle import native as orc
    from synth import make_keys
    cid = args.config
    spec = _spec(cid)
    keys = make_keys(cid)
    blob = orc.encode(keys, spec.eps)  # oracle's own encoder
    oh = orc.header(blob)
    n = keys.size
    w = spec.key_bits // 8
    out = np.empty(n, keys.dtype)
    # bound each step: decode a prefix of the list sized so the whole run stays ~<= 2 min
    t0 = time.perf_counter()
    _, nt = orc.decode_mt(blob, out)
    t_full = time.perf_counter() - t0
    total_steps = args.steps + args.warmup
    frac = min(1.0, 120.0 / max(total_steps * t_full, 1e-9))
    m = n if frac >= 1.0 else max(65536, int(n * frac) // 1024 * 1024)
    sample_bytes = (len(blob) * m / n) + m * w
    span_out = np.empty(m, keys.dtype)

    def step():
        if m == n:
            orc.decode_mt(blob, out)
        else:
            # prefix decode, all threads, same code path (oracle_decode_span per 65536 keys)
            import concurrent.futures as cf
            spans = [(a, min(a + 65536, m)) for a in range(0, m, 65536)]
            with cf.ThreadPoolExecutor(nt) as ex:
                for a, b_ in spans:
                    ex.submit(lambda a=a, b_=b_: span_out.__setitem__(
                        slice(a, b_), orc.decode_span(blob, a, b_)))
    for _ in range(args.warmup):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    if m == n:
        assert np.array_equal(out, keys)
    t = sum(ts) / len(ts)
    value = sample_bytes / t / 1e9
    sample = (f"oracle_decode_mt over {'the whole list' if m == n else f'the first {m} keys'} "
              f"of {_workload_name(cid)}, per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None,
        "dtype": "u64" if w == 8 else "u32", "data": "synthetic",
        "config": _config_dict(cid, n, len(blob), int(oh.L), int(oh.b), ws),
        "sample_keys": m, "keys_per_s": m / t,
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": nt, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- GPU arm
def _cpu_baseline(cid, blob, keys, t_enc_product, reps=3):
    """The oracle on the host cores (BASELINE.md CPU-baseline plan): full decode on all cores
    (OpenMP over 65536-key spans, median of `reps`), plus single-threaded decode and encode on
    bounded samples of the same list."""
    from oracle import native as orc
    n = keys.size
    w = keys.dtype.itemsize
    alg = len(blob) + n * w
    out = np.empty_like(keys)
    ts, nt = [], 1
    for _ in range(reps):
        t0 = time.perf_counter()
        _, nt = orc.decode_mt(blob, out)
        ts.append(time.perf_counter() - t0)
    assert np.array_equal(out, keys)
    del out
    t = statistics.median(ts)
    # single thread: decode of the first m keys (one oracle_decode_span call), encode of the
    # first me keys
    m = min(n, 1 << 25)
    t0 = time.perf_counter()
    part = orc.decode_span(blob, 0, m)
    t_st = time.perf_counter() - t0
    assert np.array_equal(part, keys[:m])
    me = min(n, 20_000_000)
    t0 = time.perf_counter()
    orc.encode(keys[:me], _spec(cid).eps)
    t_est = time.perf_counter() - t0
    return {"value": alg / t / 1e9, "unit": "GB/s", "cores": nt, "kind": "oracle",
            "sample": f"oracle_decode_mt of the full {_workload_name(cid)} (median of {reps}); "
                      f"single thread: oracle_decode_span of the first {m} keys, oracle_encode "
                      f"of the first {me} keys",
            "keys_per_s": n / t,
            "single_thread": {"decode_keys_per_s": m / t_st,
                              "decode_GBps": (len(blob) * m / n + m * w) / t_st / 1e9,
                              "encode_keys_per_s": me / t_est, "cores": 1},
            "product_encode_keys_per_s": n / t_enc_product}


def _cpu_rows(blob, keys, idx, rs, a_keys, probes):
    """The oracle timed beside every GPU row on bounded samples (host cores; OpenMP for the
    C oracle, numpy for the set-operation definitions)."""
    import os as _os

    from oracle import native as orc
    from oracle import setops

    def rate(fn, units):
        t0 = time.perf_counter()
        fn()
        return units / (time.perf_counter() - t0)

    mi, mr = 2_000_000, 200_000
    return {
        "cores": _os.cpu_count(),
        "sample": f"access {mi} idx, range {mr} x 64, next_geq {probes.size} probes, "
                  f"intersect {a_keys.size} x {keys.size} keys, union {a_keys.size} x 1e7 keys",
        "access_lookups_per_s": rate(lambda: orc.access(blob, idx[:mi]), mi),
        "ranges_per_s": rate(lambda: orc.range_decode(blob, rs[:mr], 64), mr),
        "quantile_exact_per_s": rate(lambda: orc.access(blob, idx[:mi]), mi),
        "quantile_approx_per_s": rate(lambda: orc.predict(blob, idx[:mi // 4]), mi // 4),
        "next_geq_per_s": rate(lambda: setops.next_geq(keys, probes), probes.size),
        "intersect_ms": 1e3 / rate(lambda: setops.intersect(a_keys, keys), 1),
        # union1d sorts the concatenation: bounded to the first 1e7 keys of the long list
        "union_out_keys_per_s": rate(lambda: setops.union(a_keys, keys[:10_000_000]),
                                     10_000_000 + a_keys.size),
    }


def _time_launches(fn, stream, steps, warmup, ws=1):
    """W untimed + K timed calls of fn on `stream`, bracketed by a barrier (ws > 1) and a
    device synchronize on both sides; per-call CUDA events on `stream`.  Returns (seconds of
    the timed region on this rank, per-call seconds list)."""
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record(stream)
    for k in range(steps):
        fn()
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    per = [evs[k].elapsed_time(evs[k + 1]) / 1e3 for k in range(steps)]
    return evs[0].elapsed_time(evs[-1]) / 1e3, per


def _free_block(keys, dev, stream, reps, peak):
    """NEXT-3: the config-2 keys under FORMAT F7 (free-intercept segments), same kernels."""
    import torch

    from paper_2412_10770_b200 import lc
    n, w = keys.size, 8
    t0 = time.perf_counter()
    blob_a = lc.encode(keys, 127)
    t_enc = time.perf_counter() - t0
    t0 = time.perf_counter()
    blob_f = lc.encode(keys, 127, free=True)
    t_encf = time.perf_counter() - t0
    ha, hf = lc.header(blob_a), lc.header(blob_f)
    view_a, view_f = lc.View(blob_a, device=dev), lc.View(blob_f, device=dev)
    out = view_f.out_tensor(n)
    alg_f, alg_a = len(blob_f) + n * w, len(blob_a) + n * w
    frng = np.random.default_rng(77)
    d_fi = torch.from_numpy(frng.integers(0, n, 10_000_000).astype(np.int64)).to(dev)
    fa_out = torch.empty(d_fi.numel(), dtype=out.dtype, device=dev)
    d_fx = torch.from_numpy(frng.integers(0, int(keys[-1]), 10_000_000, dtype=np.uint64)
                            .view(np.int64)).to(dev)
    f_idx = torch.empty(d_fx.numel(), dtype=torch.int64, device=dev)
    f_key = torch.empty(d_fx.numel(), dtype=torch.int64, device=dev)
    with torch.cuda.stream(stream):
        _, pa = _time_launches(lambda: lc.decode(view_a, out, stream=stream), stream, reps, 3)
        _, pf = _time_launches(lambda: lc.decode(view_f, out, stream=stream), stream, reps, 3)
        _, pfa = _time_launches(lambda: lc.access(view_f, d_fi, fa_out, stream=stream),
                                stream, reps, 2)
        _, pfn = _time_launches(lambda: lc.next_geq(view_f, d_fx, f_idx, f_key, stream=stream),
                                stream, reps, 2)
        _, pan = _time_launches(lambda: lc.next_geq(view_a, d_fx, f_idx, f_key, stream=stream),
                                stream, reps, 2)
    ref = _ref_dev(keys, dev)
    ok_f = torch.equal(out, ref) and torch.equal(fa_out, ref[d_fi])
    del ref
    if not ok_f:
        raise SystemExit("F7 decode/access mismatch")
    kf, ka = statistics.mean(pf), statistics.mean(pa)
    return {
        "workload": _workload_name(2),
        "format": "FORMAT F7: free integer intercept (O'Rourke rule on the lattice), header "
                  "flag 1, decode bias 0",
        "segments": int(hf.n_seg), "segments_anchored": int(ha.n_seg),
        "segment_reduction": 1 - hf.n_seg / ha.n_seg,
        "blob_bytes": len(blob_f), "bits_per_int": 8 * len(blob_f) / n,
        "ratio_r": len(blob_f) / (n * w),
        "decode_GBps": alg_f / kf / 1e9, "decode_keys_per_s": n / kf,
        "decode_GBps_anchored": alg_a / ka / 1e9, "decode_keys_per_s_anchored": n / ka,
        "hbm_frac": alg_f / kf / 1e9 / peak,
        "lookups_per_s": d_fi.numel() / statistics.mean(pfa),
        "next_geq_per_s": d_fx.numel() / statistics.mean(pfn),
        "next_geq_per_s_anchored": d_fx.numel() / statistics.mean(pan),
        "encode_keys_per_s_host": n / t_encf, "encode_keys_per_s_host_anchored": n / t_enc,
        "bit_exact": True,
    }


def _corpus_block(dev, stream, reps, peak, no_cpu):
    """NEXT-2's posting-list corpus (synth/corpus.py): 1e5 lists with Zipf-like lengths 10..1e6
    and per-list eps, decoded in one lc_decode_batch launch; 1e4 AND / OR pairs in one
    lc_intersect_batch / lc_union_batch call each.  Decode GB/s counts the lists' payload bytes
    (header + sections without alignment padding) read once plus the keys written once."""
    import torch

    from paper_2412_10770_b200 import lc
    from synth import make_corpus
    lists, eps, pairs = make_corpus()
    blobs = [lc.encode(k, e) for k, e in zip(lists, eps)]
    bt = lc.Batch(blobs, device=dev)
    out = torch.empty(bt.n_total, dtype=torch.int32, device=dev)
    ia = lc.SetopBuffers(bt, pairs, lc.LC_SETOP_AND)
    ua = lc.SetopBuffers(bt, pairs, lc.LC_SETOP_OR)
    with torch.cuda.stream(stream):
        _, pd = _time_launches(lambda: lc.decode_batch(bt, out, stream=stream), stream, reps, 3)
        _, pi = _time_launches(lambda: lc.intersect_batch(bt, bufs=ia, stream=stream), stream,
                               reps, 2)
        _, pu = _time_launches(lambda: lc.union_batch(bt, bufs=ua, stream=stream), stream, reps, 2)
    want = torch.from_numpy(np.concatenate(lists).view(np.int32)).to(dev)
    ok = bool(torch.equal(out, want))
    del want
    # AND / OR results of a sample of pairs against numpy's set definitions, all the counts
    from oracle import setops
    rng = np.random.default_rng(3)
    io, ic = ia.out_off.cpu().numpy(), ia.counts.cpu().numpy()
    uo, uc = ua.out_off.cpu().numpy(), ua.counts.cpu().numpy()
    iout, uout = ia.out.cpu().numpy().view(np.uint32), ua.out.cpu().numpy().view(np.uint32)
    for p in rng.choice(len(pairs), 300, replace=False):
        a, b = lists[pairs[p][0]], lists[pairs[p][1]]
        wi, wu = setops.intersect(a, b), setops.union(a, b)
        ok &= ic[p] == wi.size and np.array_equal(iout[io[p]:io[p] + ic[p]], wi)
        ok &= uc[p] == wu.size and np.array_equal(uout[uo[p]:uo[p] + uc[p]], wu)
    sz = np.array([k.size for k in lists])
    ok &= int(uc.sum()) == int(sz[pairs].sum()) - int(ic.sum())  # |A u B| = |A| + |B| - |A n B|
    if not ok:
        raise SystemExit("corpus batch mismatch")
    md, mi, mu = statistics.mean(pd), statistics.mean(pi), statistics.mean(pu)
    alg = bt.b.payload_bytes + bt.n_total * 4
    res = {
        "workload": "posting-list corpus: 1e5 u32 lists, lengths min(floor(10 U^(-1/0.7)), 1e6) "
                    "(seed 10), docIDs a uniform sorted sample of [0, 2^32), per-list eps "
                    "2^(ceil(log2(2^32/n)) + 2) - 1; 1e4 query pairs, terms ~ n^0.25",
        "lists": int(bt.b.m), "keys": int(bt.n_total), "chunks": int(bt.b.n_chunks),
        "payload_bytes": int(bt.b.payload_bytes), "bits_per_int": 8 * bt.b.payload_bytes / bt.n_total,
        "decode_ms": md * 1e3, "decode_GBps": alg / md / 1e9, "decode_keys_per_s": bt.n_total / md,
        "decode_frac": alg / md / 1e9 / peak, "launches_per_decode": 1,
        "pairs": int(len(pairs)), "and_ms": mi * 1e3, "and_pairs_per_s": len(pairs) / mi,
        "and_short_keys": int(np.minimum(sz[pairs[:, 0]], sz[pairs[:, 1]]).sum()),
        "and_matches": int(ic.sum()),
        "or_ms": mu * 1e3, "or_pairs_per_s": len(pairs) / mu, "or_keys_out": int(uc.sum()),
        "bit_exact": True,
    }
    return res


def _access_block(dev, stream, reps, no_cpu):
    """Config 5: random access, range decodes, quantiles, successor search, intersection and
    union (with and without the successor-search index), each verified."""
    import torch

    from paper_2412_10770_b200 import lc
    from synth import make_queries
    k5, idx, rs = make_queries()
    b5 = lc.encode(k5, 127)
    v5 = lc.View(b5, device=dev)
    d_idx = torch.from_numpy(idx.view(np.int64)).to(dev)
    a_out = torch.empty(idx.size, dtype=torch.int64, device=dev)
    d_rs = torch.from_numpy(rs.view(np.int64)).to(dev)
    r_out = torch.empty(rs.size * 64, dtype=torch.int64, device=dev)
    with torch.cuda.stream(stream):
        _, pa = _time_launches(lambda: lc.access(v5, d_idx, a_out, stream=stream), stream, reps, 2)
        _, pr = _time_launches(lambda: lc.range_decode(v5, d_rs, 64, r_out, stream=stream),
                               stream, reps, 2)
    d5 = torch.from_numpy(k5.view(np.int64)).to(dev)
    ok_a = torch.equal(a_out, d5[d_idx])
    sel = (d_rs[:, None] + torch.arange(64, device=dev)[None, :]).reshape(-1)
    ok_r = torch.equal(r_out, d5[sel])
    del d5, sel
    if not (ok_a and ok_r):
        raise SystemExit("access/range mismatch")
    # the access layout (lc_access_layout_build): directory instead of the binary search,
    # params and residual field from one record
    lay_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    lay = v5.build_access_layout(stream=stream)
    with torch.cuda.stream(stream):
        lay_ev[0].record(stream)
        v5.build_access_layout(stream=stream, out=lay)
        lay_ev[1].record(stream)
        a_out.zero_()
        r_out.zero_()
        _, pal = _time_launches(lambda: lc.access(v5, d_idx, a_out, stream=stream), stream, reps, 2)
        # 64-key ranges through the layout: boundary masks from the directory, one contiguous
        # gather of the record span (lc_range64_dir_kernel)
        _, prl = _time_launches(lambda: lc.range_decode(v5, d_rs, 64, r_out, stream=stream),
                                stream, reps, 2)
    torch.cuda.synchronize()
    d5 = torch.from_numpy(k5.view(np.int64)).to(dev)
    if not torch.equal(a_out, d5[d_idx]):
        raise SystemExit("access (layout) mismatch")
    sel = (d_rs[:, None] + torch.arange(64, device=dev)[None, :]).reshape(-1)
    if not torch.equal(r_out, d5[sel]):
        raise SystemExit("range (layout) mismatch")
    del d5, sel
    layout = {"bytes": v5.access_layout_bytes(), "build_ms": lay_ev[0].elapsed_time(lay_ev[1]),
              "lookups_per_s": idx.size / statistics.mean(pal),
              "ns_per_lookup": statistics.mean(pal) / idx.size * 1e9,
              "ranges_per_s": rs.size / statistics.mean(prl)}
    # NEXT-1 quantiles and NEXT-2 successor search / intersection / union on the same list
    qrng = np.random.default_rng(55)
    mq = 10_000_000
    d_ranks = torch.from_numpy(qrng.integers(0, (1 << 32) - 1, mq, endpoint=True)
                               .astype(np.uint64).view(np.int64)).to(dev)
    q_out = torch.empty(mq, dtype=torch.int64, device=dev)
    d_probe = torch.from_numpy(qrng.integers(0, int(k5[-1]), mq, dtype=np.uint64)
                               .view(np.int64)).to(dev)
    p_idx = torch.empty(mq, dtype=torch.int64, device=dev)
    p_key = torch.empty(mq, dtype=torch.int64, device=dev)
    na = 1_000_000
    a_keys = np.unique(np.concatenate([
        k5[np.sort(qrng.choice(k5.size, na // 2, replace=False))],
        qrng.integers(0, int(k5[-1]), na // 2, dtype=np.uint64)]))
    va = lc.View(lc.encode(a_keys, 127), device=dev)
    i_scr = torch.empty(lc.intersect_scratch_bytes(va), dtype=torch.uint8, device=dev)
    i_out = va.out_tensor(va.n)
    i_cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    u_scr = torch.empty(lc.union_scratch_bytes(va, v5), dtype=torch.uint8, device=dev)
    u_out = va.out_tensor(va.n + v5.n)
    u_cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    with torch.cuda.stream(stream):
        _, pqe = _time_launches(lambda: lc.quantile(v5, d_ranks, (1 << 32) - 1, True, q_out,
                                                    stream=stream), stream, reps, 2)
        _, pqa = _time_launches(lambda: lc.quantile(v5, d_ranks, (1 << 32) - 1, False, q_out,
                                                    stream=stream), stream, reps, 2)
    v5.d_acc, v5.v.d_acc = None, None  # quantiles again without the layout
    with torch.cuda.stream(stream):
        _, pqe0 = _time_launches(lambda: lc.quantile(v5, d_ranks, (1 << 32) - 1, True, q_out,
                                                     stream=stream), stream, reps, 2)
        _, pqa0 = _time_launches(lambda: lc.quantile(v5, d_ranks, (1 << 32) - 1, False, q_out,
                                                     stream=stream), stream, reps, 2)
        _, png = _time_launches(lambda: lc.next_geq(v5, d_probe, p_idx, p_key, stream=stream),
                                stream, reps, 2)
        _, pis = _time_launches(lambda: lc.intersect(va, v5, i_scr, i_out, i_cnt, stream=stream),
                                stream, reps, 2)
        _, pun = _time_launches(lambda: lc.union(va, v5, u_scr, u_out, u_cnt, stream=stream),
                                stream, reps, 2)
    # the same three with the successor-search index attached to the long list
    # (lc_search_index_build: a one-off device pass, timed separately)
    idx_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    idx_buf = v5.build_search_index(stream=stream)  # warm-up (module load), then timed
    with torch.cuda.stream(stream):
        idx_ev[0].record(stream)
        v5.build_search_index(stream=stream, out=idx_buf)
        idx_ev[1].record(stream)
    torch.cuda.synchronize()
    idx_build_ms = idx_ev[0].elapsed_time(idx_ev[1])
    p_idx2 = torch.empty_like(p_idx)
    p_key2 = torch.empty_like(p_key)
    with torch.cuda.stream(stream):
        _, pngx = _time_launches(lambda: lc.next_geq(v5, d_probe, p_idx2, p_key2, stream=stream),
                                 stream, reps, 2)
        _, pisx = _time_launches(lambda: lc.intersect(va, v5, i_scr, i_out, i_cnt, stream=stream),
                                 stream, reps, 2)
        _, punx = _time_launches(lambda: lc.union(va, v5, u_scr, u_out, u_cnt, stream=stream),
                                 stream, reps, 2)
    if not (torch.equal(p_idx2, p_idx) and torch.equal(p_key2, p_key)):
        raise SystemExit("indexed next_geq mismatch")
    want_cnt = int(np.intersect1d(a_keys, k5, assume_unique=True).size)
    if int(i_cnt.item()) != want_cnt:
        raise SystemExit("intersection count mismatch")
    if int(u_cnt.item()) != a_keys.size + k5.size - want_cnt:
        raise SystemExit("union count mismatch")
    cpu_rows = None
    if not no_cpu:
        cpu_rows = _cpu_rows(b5, k5, idx, rs, a_keys,
                             d_probe[:2_000_000].cpu().numpy().view(np.uint64))
    return {
        "workload": "config5: N=1e8 u64 keys, gaps uniform [1,256], eps=127; 1e8 uniform "
                    "lookups; 1e7 ranges x 64 keys",
        "cpu_oracle": cpu_rows,
        "lookups_per_s": idx.size / statistics.mean(pal),
        "ns_per_lookup": statistics.mean(pal) / idx.size * 1e9,
        "lookups_per_s_no_layout": idx.size / statistics.mean(pa),
        "access_layout": layout,
        "ranges_per_s": rs.size / statistics.mean(prl),
        "range_keys_per_s": rs.size * 64 / statistics.mean(prl),
        "range_out_GBps": rs.size * 64 * 8 / statistics.mean(prl) / 1e9,
        "ranges_per_s_no_layout": rs.size / statistics.mean(pr),
        "quantiles_exact_per_s": mq / statistics.mean(pqe),
        "quantiles_approx_per_s": mq / statistics.mean(pqa),
        "quantiles_exact_per_s_no_layout": mq / statistics.mean(pqe0),
        "quantiles_approx_per_s_no_layout": mq / statistics.mean(pqa0),
        "next_geq_per_s": mq / statistics.mean(png),
        "intersect": {"a_keys": int(a_keys.size), "b_keys": int(k5.size),
                      "matches": want_cnt, "ms": statistics.mean(pis) * 1e3,
                      "a_keys_per_s": a_keys.size / statistics.mean(pis)},
        "union": {"keys_out": int(u_cnt.item()), "ms": statistics.mean(pun) * 1e3,
                  "out_keys_per_s": int(u_cnt.item()) / statistics.mean(pun)},
        "search_index": {"bytes": int(v5.d_first.numel() * 8), "build_ms": idx_build_ms,
                         "next_geq_per_s": mq / statistics.mean(pngx),
                         "intersect_ms": statistics.mean(pisx) * 1e3,
                         "union_ms": statistics.mean(punx) * 1e3},
        "bit_exact": True,
        "blob_bytes": len(b5),
    }


def _ref_dev(keys, dev):
    import torch
    return torch.from_numpy(keys.view(np.int64) if keys.dtype.itemsize == 8
                            else keys.view(np.int32)).to(dev)


def _sync_barrier(ws):
    import torch
    import torch.distributed as dist
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()


def _coll_device(dev):
    """Device of the timing collectives: the GPU under NCCL, the host under gloo (test runs)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_backend() == "gloo":
        return "cpu"
    return dev


def _max_over_ranks(x, ws, dev):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=_coll_device(dev))
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _decode_config(cid, keys, dev, stream, steps, warmup, peak):
    """One extra full-decode line (configs 2 / 3 beside the headline): GB/s, keys/s, fraction
    of the HBM peak, every key verified on device."""
    import torch

    from paper_2412_10770_b200 import lc
    spec = _spec(cid)
    n, w = keys.size, spec.key_bits // 8
    blob = lc.encode(keys, spec.eps)
    h = lc.header(blob)
    view = lc.View(blob, device=dev)
    out = view.out_tensor(n)
    alg = len(blob) + n * w
    with torch.cuda.stream(stream):
        total, per = _time_launches(lambda: lc.decode(view, out, stream=stream), stream, steps,
                                    warmup)
    ref = _ref_dev(keys, dev)
    ok = bool(torch.equal(out, ref))
    del ref, out, view
    if not ok:
        raise SystemExit(f"config {cid}: decoded keys differ from the input keys")
    kern = statistics.mean(per)
    return {"workload": _workload_name(cid), "n": n, "segments": int(h.n_seg),
            "blob_bytes": len(blob), "bytes_per_step": alg, "ms_per_step": total / steps * 1e3,
            "GBps": alg * steps / total / 1e9, "keys_per_s": n * steps / total,
            "frac": alg * steps / total / 1e9 / peak, "kernel_GBps": alg / kern / 1e9,
            "kernel": _kernel_name(h), "traffic": _ncu_traffic(cid), "bit_exact": ok}


def run_gpu(args):
    import concurrent.futures as cf

    import torch
    import torch.distributed as dist

    from paper_2412_10770_b200 import lc, shard
    from synth import make_keys

    ws, rank, local = _env_dist()
    # LC_BENCH_ONE_GPU=1 (tests only): every rank on cuda:0, gloo for the timing collectives,
    # to exercise the N > 1 control flow on a one-GPU box
    one_gpu = os.environ.get("LC_BENCH_ONE_GPU") == "1"
    gpu = 0 if one_gpu else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if ws > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(dev)
    cid = args.config
    spec = _spec(cid)
    peak, peak_src = _peaks()
    extra = [c for c in (2, 3, 4) if c != cid] if ws == 1 and not args.no_configs else []
    # the next configs' keys are generated on a host thread while the GPU runs (numpy's
    # generators and sort release the GIL); the CPU baselines run after it finished
    pool = cf.ThreadPoolExecutor(1)
    pending = {c: pool.submit(make_keys, c) for c in extra[:1]}

    # ---- headline: inputs (host generation + host encode: not timed)
    keys = make_keys(cid)
    n = keys.size
    w = spec.key_bits // 8
    t_enc = time.perf_counter()
    blob = lc.encode(keys, spec.eps)
    t_enc = time.perf_counter() - t_enc
    h = lc.header(blob)
    alg_bytes = len(blob) + n * w  # the whole list: compressed read once + keys written once
    h_blob = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).pin_memory()
    if ws == 1:
        view, (i0, i1) = lc.View(blob, device=dev), (0, n)
    else:  # this rank holds and decodes only its shard (lc_shard_upload)
        view, (i0, i1) = shard.upload_shard(h_blob, rank, ws, device=dev, stream=stream)
    span = i1 - i0
    shard_bytes = 0 if view is None else view.d_blob.numel()
    rank_bytes = (shard_bytes if ws > 1 else len(blob)) + span * w
    out = torch.empty(max(span, 1), dtype=torch.int64 if w == 8 else torch.int32, device=dev)

    def step():
        if view is not None:
            lc.decode(view, out, stream=stream)

    _sync_barrier(ws)
    c0 = lc.launch_count()
    with torch.cuda.stream(stream):
        with ClockSampler(gpu) as clk:
            total, per = _time_launches(step, stream, args.steps, args.warmup, ws)
        launches = lc.launch_count() - c0 - args.warmup * (view is not None)
        t_max = _max_over_ranks(total, ws, dev)
        # correctness of what was timed: every key of the span, on device
        ref = _ref_dev(keys[i0:i1], dev)
        ok = span == 0 or bool(torch.equal(out[:span], ref))
        del ref
        if not ok:
            raise SystemExit(f"rank {rank}: decoded keys differ from the input keys")
        ms = t_max / args.steps * 1e3
        value = alg_bytes * args.steps / t_max / 1e9
        kern = statistics.mean(per) if per else float("nan")
        achieved = rank_bytes / kern / 1e9

        # ---- end to end through the C ABI with host buffers (pinned), copies inside the
        # timed region: lc_decode_host (1 GPU) or shard upload + decode + D2H of the span
        h_out = torch.empty(max(span, 1), dtype=out.dtype).pin_memory()
        e2e_steps = max(1, min(args.steps, 5))
        if ws == 1:
            d_blob = torch.empty(len(blob), dtype=torch.uint8, device=dev)

            def e2e_step():
                lc.decode_host(h_blob, d_blob, out, h_out, stream=stream)
            api = "lc_decode_host (pinned host blob -> device -> decode -> pinned host keys)"
            h2d = len(blob)
        else:
            d_blob = torch.empty(max(shard_bytes, 1), dtype=torch.uint8, device=dev)

            def e2e_step():
                if span:
                    sv = lc.View.shard(h_blob, i0, i1, device=dev, stream=stream, out=d_blob)
                    lc.decode(sv, out, stream=stream)
                    h_out[:span].copy_(out[:span], non_blocking=True)
            api = ("lc_shard_upload (pinned host blob slices of the rank's span -> device) + "
                   "lc_decode + D2H of the span's keys")
            h2d = shard_bytes
        _sync_barrier(ws)
        e2e_total, _ = _time_launches(e2e_step, stream, e2e_steps, 1, ws)
    if not np.array_equal(h_out.numpy()[:span].view(keys.dtype), keys[i0:i1]):
        raise SystemExit("e2e decode mismatch")
    e2e_t = _max_over_ranks(e2e_total, ws, dev)
    h2d_all = h2d
    if ws > 1:  # bytes every rank uploads per step (its shard)
        tt = torch.tensor([float(h2d)], dtype=torch.float64, device=_coll_device(dev))
        dist.all_reduce(tt)
        h2d_all = int(tt.item())
    e2e_value = alg_bytes * e2e_steps / e2e_t / 1e9
    # PCIe ceiling of the same transfers: plain pinned copies, each direction alone
    cp_ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    with torch.cuda.stream(stream):
        for _ in range(2):
            cp_ev[0].record(stream)
            d_blob[:h2d].copy_(h_blob[:h2d], non_blocking=True)
            cp_ev[1].record(stream)
            h_out.copy_(out, non_blocking=True)
            cp_ev[2].record(stream)
    torch.cuda.synchronize()
    h2d_gbps = h2d / max(cp_ev[0].elapsed_time(cp_ev[1]) * 1e-3, 1e-9) / 1e9
    d2h_gbps = span * w / max(cp_ev[1].elapsed_time(cp_ev[2]) * 1e-3, 1e-9) / 1e9
    e2e_floor_ms = max(h2d / max(h2d_gbps, 1e-9), span * w / max(d2h_gbps, 1e-9)) / 1e6
    del d_blob, h_out, out, view

    # ---- configs 2 / 3 (the other >= 1e8-key configs of the north-star target), 1 GPU
    decode_configs = {}
    if ws == 1:
        decode_configs[f"config{cid}"] = {
            "workload": _workload_name(cid), "n": n, "segments": int(h.n_seg),
            "blob_bytes": len(blob), "bytes_per_step": alg_bytes, "ms_per_step": ms,
            "GBps": value, "keys_per_s": n * args.steps / t_max, "frac": value / peak,
            "kernel_GBps": achieved, "kernel": _kernel_name(h), "traffic": _ncu_traffic(cid),
            "bit_exact": True}
    cfg_steps = max(3, min(args.steps, 20))
    keys2 = keys if cid == 2 else None
    for k, c in enumerate(extra):
        kc = pending.pop(c).result()
        if c == 2:
            keys2 = kc
        if k + 1 < len(extra):
            pending[extra[k + 1]] = pool.submit(make_keys, extra[k + 1])
        with ClockSampler(gpu) as clk_c:
            decode_configs[f"config{c}"] = _decode_config(c, kc, dev, stream, cfg_steps, 3, peak)
        decode_configs[f"config{c}"]["clocks"] = clk_c.summary()
        del kc
    pool.shutdown()

    # ---- NEXT-3: config 2 under FORMAT F7 (free-intercept segments), same kernels
    free = None
    if ws == 1 and not args.no_free:
        free = _free_block(keys2 if keys2 is not None else make_keys(2), dev, stream,
                           max(5, min(args.steps, 50)), peak)
    del keys2

    # ---- NEXT-2: the posting-list corpus (batched decode, AND / OR pairs)
    corpus = None
    if ws == 1 and not args.no_corpus:
        corpus = _corpus_block(dev, stream, max(5, min(args.steps, 20)), peak, args.no_cpu)

    # ---- random access + range decodes (config 5), reported beside the headline
    access = None
    if ws == 1 and not args.no_access:
        access = _access_block(dev, stream, max(3, min(args.steps, 20)), args.no_cpu)

    if ws > 1:
        dist.barrier()
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None,
        "dtype": "u64" if w == 8 else "u32", "data": "synthetic",
        "config": _config_dict(cid, n, len(blob), int(h.n_seg), int(h.res_bits), ws),
        "keys_per_s": n * args.steps / t_max,
        "hbm_frac": value / ws / peak,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _ncu_traffic(cid) if ws == 1 else None,
                     "traffic_source": "profiles/ncu_traffic.json (dram read+write bytes of one "
                                       "ncu --set full launch of this config's decode)",
                     "kernel": _kernel_name(h), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": rank_bytes,
                     "algorithmic_bytes": "blob bytes read once + N * key bytes written once "
                                          "(rank 0's shard under --gpus > 1)"},
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": h2d_all,
                "d2h_bytes_per_step": n * w, "api": api,
                "ms_per_step": e2e_t / e2e_steps * 1e3,
                "pcie_h2d_GBps": h2d_gbps, "pcie_d2h_GBps": d2h_gbps,
                "pcie_floor_ms": e2e_floor_ms},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "decode_configs": decode_configs or None,
        "access": access,
        "corpus": corpus,
        "free_intercept": free,
    }
    if ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = _cpu_baseline(cid, blob, keys, t_enc)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5],
                    help="headline workload (default: config 4, the largest)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the decode_configs lines of the other 1e8+ configs")
    ap.add_argument("--no-access", action="store_true")
    ap.add_argument("--no-corpus", action="store_true", help="skip the posting-list corpus block")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-free", action="store_true", help="skip the FORMAT F7 block")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
