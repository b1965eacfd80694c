#!/usr/bin/env python
"""Benchmark of the Huskysort hot path on B200 (BASELINE.json metric: strings
sorted/sec at 1/2/4/8 B200; radix/encode HBM GB/s vs peak).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C5] [--n N] [--no-also] [--no-cpu-baseline]

A step = one full sort (encode -> onesweep radix -> gather + run detection /
order check -> fix-up) of one batch of synthetic strings through the C ABI,
inputs already resident in HBM.  The headline workload is BASELINE.json's
metric configuration C5: ONE dataset of 2^30 ASCII strings (len U[8,24],
[0-9A-Za-z], ~1% duplicates, first 10% pre-sorted), generated block-wise on
the device (workloads/gen.cu).  N = 1 sorts all of it with husky_sort; N > 1
(torchrun, one rank per GPU) shards the SAME dataset -- rank r holds block
[r*N/P, (r+1)*N/P) -- and runs the NCCL sample sort (strong scaling).  Every
timed output is validated on the device with the linear verifier (checker/).
Rank 0 prints ONE JSON line; secondary workloads (C2 at N = 1, C4 at N > 1)
ride in its "also" object.  `--impl reference` times the CPU oracle (the
reference arm of this tier: the paper has no code) on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "strings sorted/sec (M/s) at 1/2/4/8 B200; radix/encode HBM GB/s vs peak"
UNIT = "Mstrings/s"
DESCR = {
    "C1": "C1: 1e5 lowercase a-z strings, len U[4,12], ASCII coder",
    "C2": "C2: 1e7 English-like words, Zipf(1.0) over a 50,000-word synthetic vocabulary, ASCII coder",
    "C3": "C3: 1e7 UTF-16 CJK strings (U+4E00-U+9FFF), len U[2,4], UNICODE coder",
    "C4": "C4: 1e7 ASCII strings sharing a 16-char prefix + 8 random [0-9A-Za-z] (all codes collide)",
    "C5": "C5: 2^30 ASCII strings, len U[8,24], [0-9A-Za-z], ~1% exact duplicates, first 10% pre-sorted "
          "(one dataset; block-wise counter generator)",
    "D1": "D1 (fix-up workload, not a BASELINE config): 1e7 ASCII strings in shuffled groups of U[100,4096] "
          "sharing a 12-char prefix (one dirty equal-code run per group) + 1..10 random a-z",
}
# random reads past ~2 GB are capped at ~36 G accesses/s for 16-64 B blocks
# (profiles/r02_random_access_probe.txt): the gather's second roofline
RANDOM_ACCESS_PEAK = 36.0e9
PACK_MAX_N = 1 << 28
SLAB_MAX = {0: 24, 1: 10}   # units a slab record covers (ASCII / UNICODE)
PL = {0: 9, 1: 3, 2: 12, 3: 10}
KWIN = {0: 9, 1: 4, 2: 12, 3: 10}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None
        self.out = ""

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            time.sleep(0.15)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), f[5], f[6], f[7], f[8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        reasons = set()
        for r in rows:
            for nm, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], r[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


def cpu_info():
    try:
        nproc = len(os.sched_getaffinity(0))
    except Exception:
        nproc = os.cpu_count() or 1
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return nproc, model


# ----------------------------------------------------------------- CPU legs
def host_workload(name, n):
    return W.c5(n) if name == "C5" else W.make(name, n)


def cpu_baseline(name, n_sample):
    """The oracle as it stands, on the host cores: the single-threaded merge sort
    (T = 1) and the T = nproc chunk-sort + pairwise-merge variant, on a bounded
    sample of the same workload recipe."""
    import oracle
    oracle.build()
    nproc, model = cpu_info()
    w = host_workload(name, n_sample)

    def timed(fn, min_s, max_calls):
        calls, dt, out = 0, 0.0, None
        while calls < max_calls and (calls == 0 or dt < min_s):
            t0 = time.perf_counter()
            out = fn()
            dt += time.perf_counter() - t0
            calls += 1
        return out, calls, dt

    p1, c1, d1 = timed(lambda: oracle.sort(w.coder, w.units, w.offsets), 6.0, 4)
    pn, cn, dn = timed(lambda: oracle.sort_mt(w.coder, w.units, w.offsets, nproc), 3.0, 8)
    assert np.array_equal(p1, pn), "T-thread oracle disagrees with the 1-thread oracle"
    recipe = (f"{name} recipe at n={n_sample} (the same generator with N = n: same length / alphabet / "
              f"duplicate / pre-sorted structure)")
    v1, vn = n_sample * c1 / d1 / 1e6, n_sample * cn / dn / 1e6
    return {"value": round(vn, 4), "unit": UNIT, "cores": nproc, "kind": "oracle",
            "sample": f"{recipe}; T={nproc}: {cn} oracle_sort_mt calls, {dn:.2f} s wall",
            "threads": nproc, "cpu_model": model,
            "t1": {"value": round(v1, 4), "unit": UNIT, "cores": 1,
                   "sample": f"{recipe}; {c1} oracle_sort calls (top-down merge sort, 1 thread), {d1:.2f} s wall"}}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    n_sample = args.ref_sample
    w = host_workload(args.config, n_sample)
    nproc, model = cpu_info()
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.sort_mt(w.coder, w.units, w.offsets, nproc)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = statistics.median(times)
    value = n_sample / t / 1e6
    sample = (f"{args.config} recipe at n={n_sample} strings per step (bounded sample of the "
              f"{W.FULL_N[args.config]}-string workload), oracle_sort_mt with {nproc} threads")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u16" if w.coder == 1 else "u8", "data": "synthetic",
            "config": {"workload": DESCR[args.config], "n_total": W.FULL_N[args.config], "sample_n": n_sample},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": nproc, "kind": "oracle",
                             "sample": sample, "cpu_model": model},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU side
def device_workload(name, n_total, base, n_local, dev):
    """Block [base, base + n_local) of the n_total-string dataset `name`, in HBM."""
    import torch
    if name == "C5":
        import workloads.gpu as G
        units, off = G.c5_device(n_total, base, n_local, dev)
        coder = 0
    else:
        w = W.make(name, n_total)
        o = w.offsets
        u = w.units[o[base]:o[base + n_local]]
        coder = w.coder
        if u.dtype == np.uint16:
            u = u.view(np.int16)
        units = torch.from_numpy(np.ascontiguousarray(np.concatenate([u, np.zeros(16, u.dtype)]))).to(dev)
        off = torch.from_numpy(o[base:base + n_local + 1] - o[base]).to(dev)
    lens = (off[1:] - off[:-1])
    ub = 2 if coder == 1 else 1
    k = KWIN[coder]
    stats = {"p_bar": float(lens.clamp(max=k).double().mean().item()),
             "l_bar": float(lens.double().mean().item()),
             "f_le_pl": float((lens <= PL[coder]).double().mean().item()),
             "f_le_slab": float((lens <= SLAB_MAX.get(coder, 0)).double().mean().item()),
             "l_bar_gt_slab": float((lens * (lens > SLAB_MAX.get(coder, 0))).double().mean().item())}
    total = int(off[-1].item())
    return {"name": name, "coder": coder, "units": units, "offsets": off, "n": n_local, "ub": ub,
            "total_units": total, "stats": stats}


def byte_models(wl, passes, packed):
    """Algorithmic bytes per string of each kernel: SURVEY.md 8(d)'s model, and
    the builder's model of what this implementation actually moves."""
    st, ub = wl["stats"], wl["ub"]
    p_bar, l_bar = st["p_bar"], st["l_bar"]
    slab = wl["coder"] in (0, 1)
    # survey 8(d): K1 = 8 + w p + 8; K3 = 24 per pass (pass 0 reads no payload: 20);
    # hist (fused in the survey's K1) = 8; K5 = 4 + 16 + 2 w l + 8
    survey = {"encode": 8 + ub * p_bar + 8, "hist": 8.0,
              "radix_pass": (20 + 24 * (passes - 1)) / passes if passes else 0.0,
              "radix_pass_first": 20.0, "radix_pass_rest": 24.0,
              "gather": 4 + 16 + 2 * ub * l_bar + 8}
    # builder: encode adds the packed payload (n <= 2^28) and the slab records
    # (every string's when not packed, else those longer than PL); pass 0 reads
    # the packed payload; the gather reads perm 4 + sorted code 8, a slab record
    # (16) or offsets (16) + units for the strings it cannot rebuild from the code
    f_dec = st["f_le_pl"] if packed else 0.0
    f_slab = (st["f_le_slab"] - f_dec) if slab else 0.0
    f_off = 1.0 - f_dec - f_slab
    l_off = st["l_bar_gt_slab"] if slab else l_bar
    builder = {"encode": survey["encode"] + (4 if packed else 0) + 16 * (st["f_le_slab"] - (f_dec if packed else 0))
               * (1 if slab else 0),
               "hist": 8.0,
               "radix_pass": ((24 if packed else 20) + 24 * (passes - 1)) / passes if passes else 0.0,
               "gather": 4 + 8 + 16 * f_slab + 16 * f_off + ub * l_off + ub * l_bar + 8}
    # random accesses per string in the gather (a 16-B slab read: 1; offsets +
    # units: 1.25 + ~1.5 for a short string)
    rand = f_slab * 1.0 + f_off * 2.75
    return survey, builder, {"f_decoded": f_dec, "f_slab": f_slab, "f_offsets": f_off, "random_per_string": rand}


def kernel_entry(name, ms_per_launch, bytes_per_launch, peak, extra=None):
    a = bytes_per_launch / (ms_per_launch * 1e-3) / 1e9 if ms_per_launch else 0.0
    d = {"kernel": name, "bound": "hbm", "achieved": round(a, 1), "peak": peak, "unit": "GB/s",
         "frac": round(a / peak, 4), "ms_per_launch": round(ms_per_launch, 5),
         "bytes_alg_per_launch": int(bytes_per_launch)}
    if extra:
        d.update(extra)
    return d


def traffic_of(config, kernel, n):
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        td = json.load(open(tp)).get(config, {}).get(kernel)
        return int(td["bytes_per_key"] * n) if td else None
    except Exception:
        return None


def measure_single(args, name, n, dev, steps, warmup, flush, want_e2e, h, torch):
    """One GPU: husky_sort of the whole dataset, K timed steps."""
    import checker
    wl = device_workload(name, n, 0, n, dev)
    coder, u, o = wl["coder"], wl["units"], wl["offsets"]
    total = wl["total_units"]
    ws = torch.empty(h.husky_sort_workspace(coder, n, total), dtype=torch.uint8, device=dev)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    su = torch.empty(total + 16, dtype=u.dtype, device=dev)
    so = torch.empty(n + 1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        outc = h.husky_sort(coder, u, o, perm, su, so, ws)
    torch.cuda.synchronize()

    # ---- timed region: K steps, an event pair per step; profiler mode 2 adds
    # event pairs around the encoder, histogram, radix-pass group and main gather
    # (large inputs only: below 2^22 strings the extra records would show in the
    # step time and they also turn off the library's CUDA-graph replay; the
    # per-kernel times then come from the breakdown steps)
    h.husky_profile_reset()
    group_events = n >= (1 << 22)
    h.husky_profile_enable(2 if group_events else 0)
    l0 = h.husky_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    bad = {"pairs": 0, "perm": 0, "content": 0, "offsets": 0}
    torch.cuda.synchronize()
    launches = 0
    with ClockSampler(dev.index or 0) as clk:
        for i in range(steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            outc = h.husky_sort(coder, u, o, perm, su, so, ws)
            ev[i][1].record(stream)
            launches += h.husky_launch_count() - l0
            # validation of this step's output, outside its events
            r = checker.verify(u, o, perm, su[:total], so)
            for k in bad:
                bad[k] += r[k]
            l0 = h.husky_launch_count()
        torch.cuda.synchronize()
    h.husky_profile_enable(False)
    groups = h.husky_profile_read() if group_events else None
    times = [a.elapsed_time(b) for a, b in ev]
    med, mn, mean = statistics.median(times), min(times), statistics.mean(times)

    # ---- per-launch breakdown (separate steps, an event pair per launch)
    h.husky_profile_reset()
    h.husky_profile_enable(1)
    n_bd = 2
    for i in range(n_bd):
        flush.fill_(i & 0xFF)
        h.husky_sort(coder, u, o, perm, su, so, ws)
    torch.cuda.synchronize()
    h.husky_profile_enable(False)
    log = h.husky_profile_launches()
    stages = {}
    for st_name, _, ms in log:
        e = stages.setdefault(st_name, {"ms_per_step": 0.0, "launches_per_step": 0})
        e["ms_per_step"] += ms / n_bd
        e["launches_per_step"] += 1 / n_bd
    for e in stages.values():
        e["ms_per_step"] = round(e["ms_per_step"], 4)
    # the main key sort's passes (refinement passes of A6 are extra and counted
    # in outcome.radix_passes; keys_partitioned counts the main sort only)
    passes = int(outc["keys_partitioned"]) // n if n else 0
    radix_launch_ms = [ms for st_name, el, ms in log if st_name == "radix_pass" and el == n]
    per_step = len(radix_launch_ms) // n_bd if n_bd else 0
    per_pass = [statistics.mean(radix_launch_ms[s * per_step + p] for s in range(n_bd)) for p in range(per_step)]
    per_pass = [t for t in per_pass][:passes]

    # ---- roofline (timed-region group events)
    peak, peak_src = peaks()
    packed = n <= PACK_MAX_N and coder in (0, 1)
    survey, builder, gstats = byte_models(wl, passes, packed)
    if groups is not None:
        g = {k: v["ms"] / steps for k, v in groups.items() if v["ms"]}
    else:  # small inputs: per-kernel times from the breakdown steps
        g = {k: v["ms_per_step"] for k, v in stages.items()}
    kern = {}
    if passes and outc["refine_rounds"] == 0:
        rp = g.get("radix_pass", 0.0) / passes
        kern["radix_pass"] = kernel_entry("k_onesweep (A2 radix pass)", rp, survey["radix_pass"] * n, peak, {
            "passes_per_sort": passes,
            "model_builder": {"bytes_alg_per_launch": int(builder["radix_pass"] * n),
                              "frac": round(builder["radix_pass"] * n / (rp * 1e-3) / 1e9 / peak, 4)},
            "per_pass": [{"pass": p, "ms": round(t, 4),
                          "frac_survey": round((20 if p == 0 else 24) * n / (t * 1e-3) / 1e9 / peak, 4)}
                         for p, t in enumerate(per_pass)],
            "per_pass_timing": "breakdown steps, an event pair per launch (outside the timed region)"})
    if g.get("encode"):
        kern["encode"] = kernel_entry("k_encode (A1)", g["encode"], survey["encode"] * n, peak, {
            "model_builder": {"bytes_alg_per_launch": int(builder["encode"] * n),
                              "frac": round(builder["encode"] * n / (g["encode"] * 1e-3) / 1e9 / peak, 4)}})
    if g.get("hist_scan"):
        kern["hist"] = kernel_entry("k_hist_slots (A2 digit histograms + plan)", g["hist_scan"], 8 * n, peak)
    if g.get("gather") and outc["refine_rounds"] == 0:  # (C4: the main gather only records the one run)
        ra = gstats["random_per_string"] * n / (g["gather"] * 1e-3)
        kern["gather"] = kernel_entry("k_gather (A4 + A3)", g["gather"], survey["gather"] * n, peak, {
            "model_builder": {"bytes_alg_per_launch": int(builder["gather"] * n),
                              "frac": round(builder["gather"] * n / (g["gather"] * 1e-3) / 1e9 / peak, 4)},
            "random_access": {"per_string": round(gstats["random_per_string"], 3),
                              "achieved_per_s": round(ra / 1e9, 2), "peak_per_s": RANDOM_ACCESS_PEAK / 1e9,
                              "unit": "G accesses/s", "frac": round(ra / RANDOM_ACCESS_PEAK, 4),
                              "peak_source": "profiles/r02_random_access_probe.txt (random 16-64 B reads "
                                             "over >= 2 GB, one B200)"},
            "strings": {k: round(v, 4) for k, v in gstats.items()}})
    for k, v in kern.items():  # DRAM bytes per launch from the committed ncu capture (profiles/traffic.json)
        v["traffic"] = traffic_of(name, k, n)
    total_ms = sum(v["ms_per_launch"] * (passes if k == "radix_pass" else 1) for k, v in kern.items())
    dom = max(kern, key=lambda k: kern[k]["ms_per_launch"] * (passes if k == "radix_pass" else 1)) if kern else None
    roof = dict(kern[dom]) if dom else {}
    if dom:
        roof.update({"traffic": traffic_of(name, dom, n), "peak_source": peak_src,
                     "share_of_step": round(kern[dom]["ms_per_launch"] * (passes if dom == "radix_pass" else 1)
                                            / med, 4),
                     "model": "survey (SURVEY.md 8(d)); model_builder beside it",
                     "timing": ("CUDA events recorded by the library on its launch stream around the kernel "
                                "group, every timed step (profiler mode 2)") if groups is not None else
                               "breakdown steps, an event pair per launch (n < 2^22: kept out of the timed steps)",
                     "kernels": kern})
    # ---- perm-only mode (no sorted strings: the run scan replaces the gather;
    # SURVEY.md 8(d) reports it separately); its perm must equal the full sort's
    del su, so
    po = torch.empty_like(perm)
    for _ in range(2):
        h.husky_sort(coder, u, o, po, None, None, ws)
    tpo = []
    for i in range(min(steps, 5)):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        h.husky_sort(coder, u, o, po, None, None, ws)
        b.record(stream)
        torch.cuda.synchronize()
        tpo.append(a.elapsed_time(b))
    mpo = statistics.median(tpo)
    perm_only = {"value": round(n / (mpo * 1e-3) / 1e6, 4), "unit": UNIT, "ms_per_step": round(mpo, 4),
                 "ms_min": round(min(tpo), 4), "steps": len(tpo),
                 "matches_full_sort_perm": bool(torch.equal(po, perm))}
    del po
    res = {"name": name, "n": n, "coder": coder, "wl": wl, "times": times, "median": med, "min": mn, "mean": mean,
           "outcome": outc, "validation": bad, "launches": launches // max(steps, 1), "stages": stages,
           "roofline": roof, "clocks": clk.summary(), "kernels_ms_sum": total_ms, "packed": packed,
           "perm_only": perm_only}
    # keep what the e2e / library legs need, drop the rest
    del ws
    res["perm_dev"] = perm
    return res


def cub_bar(h, torch, wl, steps, flush):
    """cub::DeviceRadixSort::SortPairs<u64, u32> on the same codes (bits [0, 63))."""
    lib_path = os.path.join(ROOT, "tools", "libcubbar.so")
    if not os.path.exists(lib_path):
        return None
    lib = ctypes.CDLL(lib_path)
    lib.cub_sortpairs_temp.argtypes = [ctypes.c_uint64, ctypes.POINTER(ctypes.c_size_t)]
    lib.cub_sortpairs.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                                          ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    n = wl["n"]
    codes, _ = h.husky_encode(wl["coder"], wl["units"], wl["offsets"], want_perfect=False)
    kout = torch.empty_like(codes)
    vin = torch.arange(n, dtype=torch.int32, device=codes.device)
    vout = torch.empty_like(vin)
    tb = ctypes.c_size_t(0)
    lib.cub_sortpairs_temp(n, ctypes.byref(tb))
    temp = torch.empty(tb.value, dtype=torch.uint8, device=codes.device)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ts = []
    for i in range(steps + 2):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = lib.cub_sortpairs(codes.data_ptr(), kout.data_ptr(), vin.data_ptr(), vout.data_ptr(), n, 0, 63,
                               temp.data_ptr(), tb.value, s)
        b.record()
        torch.cuda.synchronize()
        if rc:
            return {"error": f"cub rc={rc}"}
        if i >= 2:
            ts.append(a.elapsed_time(b))
    del codes, kout, vin, vout, temp
    return {"cub_sortpairs_u64_u32_ms": round(statistics.median(ts), 4), "bits": "[0, 63)",
            "what": "cub::DeviceRadixSort::SortPairs<uint64_t, uint32_t> (CUB of CUDA 12.9) on the same husky "
                    "codes, 12 B per key and pass; compare with stages.hist_scan + stages.radix_pass"}


def e2e_single(h, torch, wl, steps, warmup, dev):
    """The same metric through the C ABI with HOST buffers: every step copies
    the inputs from pinned host memory and the outputs (perm, sorted units,
    sorted offsets) back, inside the timed region."""
    coder, n, total, ub = wl["coder"], wl["n"], wl["total_units"], wl["ub"]
    dt = wl["units"].dtype
    hu = torch.empty(total + 16, dtype=dt).pin_memory()
    hu.copy_(wl["units"][:total + 16])
    ho = wl["offsets"].cpu().pin_memory()
    h2d = total * ub + (n + 1) * 8
    d2h = n * 4 + total * ub + (n + 1) * 8
    wl["units"] = wl["offsets"] = None
    torch.cuda.empty_cache()
    # pipelined: the K steps as K batches of husky_sort_host_many, H2D / kernels
    # / D2H on three streams.  Up to 2^28 strings: 2 input slots (a batch's
    # copies overlap another batch's kernels).  Above (C5: inputs + workspace
    # ~74 GB per input slot, outputs ~30 GB per output slot): ONE input slot and
    # two output slots (134 GB) -- the next batch's inputs go in over PCIe while
    # this batch's outputs come out (full duplex), and the next sort no longer
    # waits for the copy-out
    depth = 2 if n <= PACK_MAX_N else 1
    mws = torch.empty(h.husky_sort_host_many_workspace(coder, n, total, depth), dtype=torch.uint8, device=dev)
    outs = [(torch.empty(n, dtype=torch.int32).pin_memory(), torch.empty(total + 8, dtype=dt).pin_memory(),
             torch.empty(n + 1, dtype=torch.int64).pin_memory()) for _ in range(depth)]
    batches = [(hu, ho, outs[b % depth][0], outs[b % depth][1], outs[b % depth][2]) for b in range(steps)]
    h.husky_sort_host_many(coder, batches[:max(depth, warmup)], mws, depth)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.husky_sort_host_many(coder, batches, mws, depth)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    api = (f"husky_sort_host_many: {steps} steps as {steps} pipelined batches, {depth} input / {depth + 1} output "
           "device slot(s), H2D / "
           "kernels / D2H on three streams (pinned host buffers), host wall clock around the call")
    hp = outs[(steps - 1) % depth][0]
    del mws
    return {"value": round(n / (ms * 1e-3) / 1e6, 4), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3), "api": api}, hp


def run_single(args, h, torch, dev):
    name = args.config
    n = args.n or W.FULL_N[name]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    r = measure_single(args, name, n, dev, args.steps, args.warmup, flush, True, h, torch)
    wl = r["wl"]
    # library bar on the same codes
    bar = None
    if not args.no_library_bar:
        try:
            bar = cub_bar(h, torch, wl, min(args.steps, 5), flush)
            if bar and "stages" in r:
                ours = sum(r["stages"].get(k, {}).get("ms_per_step", 0.0) for k in ("hist_scan", "radix_pass"))
                bar["ours_key_sort_ms"] = round(ours, 4)
        except Exception as e:  # the bar is context; never fail the line on it
            bar = {"error": str(e)[:200]}
    # end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        perm_dev = r.pop("perm_dev").cpu()
        try:
            e2e, hp = e2e_single(h, torch, wl, args.e2e_steps, 1, dev)
            e2e["matches_device_perm"] = bool(torch.equal(hp[:n], perm_dev))
        except (RuntimeError, MemoryError, h.HuskyError) as e:  # e.g. less free HBM on the box: keep the line
            torch.cuda.empty_cache()
            e2e = {"value": None, "unit": UNIT, "error": str(e)[:200]}
    else:
        r.pop("perm_dev", None)
    del wl
    r.pop("wl", None)
    torch.cuda.empty_cache()
    also = {}
    if not args.no_also and name == "C5":
        # the other single-GPU configs (parity / structure cases of BASELINE.json)
        # and D1, a dirty-run workload that exercises the segmented fix-up (A5)
        for cfg in ("C1", "C2", "C3", "C4", "D1"):
            r2 = measure_single(args, cfg, W.FULL_N[cfg], dev, max(3, args.steps // 2), args.warmup, flush, False, h,
                                torch)
            r2.pop("perm_dev", None)
            wl2 = r2.pop("wl", None)
            rr = r2["roofline"]
            entry = {"workload": DESCR[cfg], "n": r2["n"], "value": round(r2["n"] / (r2["median"] * 1e-3) / 1e6, 4),
                     "unit": UNIT, "ms_per_step": round(r2["median"], 4), "ms_min": round(r2["min"], 4),
                     "validation": r2["validation"], "stages": r2["stages"],
                     "roofline": {k: {"frac": v["frac"], "ms_per_launch": v["ms_per_launch"],
                                      **({"per_pass": v["per_pass"]} if "per_pass" in v else {}),
                                      **({"model_builder": v["model_builder"]} if "model_builder" in v else {}),
                                      **({"random_access": v["random_access"]} if "random_access" in v else {})}
                                  for k, v in rr.get("kernels", {}).items()},
                     "outcome": r2["outcome"], "perm_only": r2["perm_only"]}
            fx = r2["stages"].get("fix_medium", {}).get("ms_per_step", 0.0) + \
                r2["stages"].get("fix_small", {}).get("ms_per_step", 0.0)
            if cfg == "D1" and fx and wl2 is not None:
                # sum over strings in runs of (w len + 8) bytes
                fb = r2["outcome"]["n_in_runs"] * (wl2["ub"] * wl2["stats"]["l_bar"] + 8)
                peak, _ = peaks()
                entry["fixup"] = {"kernels": "k_fix_staged (+ k_fix_small / k_fix_medium / k_regather_runs for runs "
                                             "that do not fit the stage)", "ms": round(fx, 4),
                                  "bytes_alg": int(fb), "achieved_gbs": round(fb / (fx * 1e-3) / 1e9, 1),
                                  "frac": round(fb / (fx * 1e-3) / 1e9 / peak, 4),
                                  "note": "the byte model is a lower bound: sorting a run of ~2000 strings costs "
                                          "O(n log n) shared-memory comparisons, not a pass over its bytes"}
            also[cfg] = entry
            del wl2
            torch.cuda.empty_cache()
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(name, min(n, args.cpu_sample))
    line = {"metric": METRIC, "value": round(n / (r["median"] * 1e-3) / 1e6, 4), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["median"], 4),
            "ms_min": round(r["min"], 4), "ms_mean": round(r["mean"], 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u16" if r["coder"] == 1 else "u8",
            "data": "synthetic",
            "config": {"workload": DESCR[name], "n_total": n, "n_per_gpu": n,
                       "coder": "unicode" if r["coder"] == 1 else "ascii",
                       "outputs": "perm + sorted units + sorted offsets",
                       "l2": "inputs > L2; a 256 MiB buffer is also written between timed steps (outside the step "
                             "events)",
                       "parallelism": "1 GPU", "timing": "median of the steps' CUDA-event times (min and mean beside)"},
            "roofline": r["roofline"], "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": r["launches"],
            "clocks": r["clocks"], "stages": r["stages"], "validation": dict(r["validation"], steps=args.steps,
                                                                             verifier="checker/verify.cu"),
            "library_bar": bar, "outcome": r["outcome"], "perm_only": r["perm_only"], "also": also or None}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ N > 1
def run_sharded(args, h, torch, dev, rank, world):
    import torch.distributed as dist

    import checker
    name = args.config
    n_total = args.n or W.FULL_N[name]
    comm = h.multi.comm_from_process_group(device=dev) if world > 1 else h.husky_comm_create(
        0, 1, h.husky_comm_unique_id())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def one(cname, n_tot, steps, warmup, want_e2e):
        base = rank * n_tot // world
        n_loc = (rank + 1) * n_tot // world - base
        wl = device_workload(cname, n_tot, base, n_loc, dev)
        coder, u, o = wl["coder"], wl["units"], wl["offsets"]
        in_hash = checker.hash_sum(u, o, gbase=base)
        outs = []
        stream = torch.cuda.current_stream()
        for _ in range(warmup):
            outs = h.sort_multi(comm, coder, u, o, base)
        torch.cuda.synchronize()
        times, bad_pairs, hash_ok = [], 0, True
        dist.barrier() if world > 1 else None
        torch.cuda.synchronize()
        launches = 0
        with ClockSampler(dev.index or 0) as clk:
            for i in range(steps):
                flush.fill_(i & 0xFF)
                if world > 1:
                    dist.barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                l0 = h.husky_launch_count()
                a.record(stream)
                outs = h.sort_multi(comm, coder, u, o, base)
                b.record(stream)
                launches += h.husky_launch_count() - l0
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
                # validation: pairs inside the shard, order across shard
                # boundaries, (gidx, string) multiset via hash sums
                p, su, so, outc = outs
                bad_pairs += checker.shard_pairs(p, su, so)
                out_hash = checker.hash_sum(su, so, perm=p)
                hs = torch.stack([in_hash, out_hash]).view(-1)
                if world > 1:
                    dist.all_reduce(hs)
                hash_ok &= int(hs[0].item()) == int(hs[1].item())
        # per-step max over ranks
        tt = torch.tensor(times, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        times = tt.cpu().tolist()
        # phase breakdown of this rank: one more step with an event pair per launch
        h.husky_profile_reset()
        h.husky_profile_enable(1)
        h.sort_multi(comm, coder, u, o, base)
        torch.cuda.synchronize()
        h.husky_profile_enable(False)
        stages = {}
        plog = h.husky_profile_launches()
        for st_name, _, ms in plog:
            e = stages.setdefault(st_name, {"ms": 0.0, "launches": 0})
            e["ms"] = round(e["ms"] + ms, 4)
            e["launches"] += 1
        p, su, so, outc = outs
        # roofline of the dominant kernel, the local sort's radix pass (this
        # rank's received strings), from the profiled step's per-launch times
        n_out = int(p.numel())
        rp = [ms for st_name, el, ms in plog if st_name == "radix_pass" and el == n_out and n_out > 0]
        passes = int(outc["keys_partitioned"]) // n_out if n_out else 0
        rp = rp[:passes]
        roof = None
        if rp:
            peak, peak_src = peaks()
            t = statistics.mean(rp)
            bytes_alg = 24 * n_out
            roof = {"kernel": "k_onesweep (A2 radix pass, local sort of rank 0)", "bound": "hbm",
                    "achieved": round(bytes_alg / (t * 1e-3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(bytes_alg / (t * 1e-3) / 1e9 / peak, 4), "traffic": None,
                    "ms_per_launch": round(t, 4), "passes_per_sort": passes, "peak_source": peak_src,
                    "timing": "profiled step (an event pair per launch), outside the timed steps"}
        # boundary check: this shard's last string < the next shard's first
        ends = [None, None]
        if p.numel():
            f0, f1 = int(so[0].item()), int(so[1].item())
            l0, l1 = int(so[-2].item()), int(so[-1].item())
            ends = [(su[f0:f1].cpu().numpy().tobytes(), int(p[0].item()) & 0xFFFFFFFF),
                    (su[l0:l1].cpu().numpy().tobytes(), int(p[-1].item()) & 0xFFFFFFFF)]
        allends = [None] * world
        if world > 1:
            dist.all_gather_object(allends, ends)
        else:
            allends = [ends]
        boundary_bad = 0
        prev = None
        for e in allends:
            if e[0] is None:
                continue
            if prev is not None and not (prev[0] < e[0][0] or (prev[0] == e[0][0] and prev[1] < e[0][1])):
                boundary_bad += 1
            prev = e[1]
        bp = torch.tensor([bad_pairs], device=dev)
        to = torch.tensor([outc["bytes_to_peers"]], dtype=torch.float64, device=dev)
        # the exchange kernel (the partition-order gather storing into the
        # peers' windows): the profiled step's "multi" launch over the n_loc
        # local strings; bandwidth = this rank's bytes to peers / its time
        xch = [ms for st_name, el, ms in plog if st_name == "multi" and el == n_loc and n_loc > 0]
        xms = float(xch[0]) if xch else 0.0
        xgbs = torch.tensor([outc["bytes_to_peers"] / (xms * 1e-3) / 1e9 if xms > 0 else 0.0, xms],
                            dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(bp)
            dist.all_reduce(to, op=dist.ReduceOp.MAX)
            dist.all_reduce(xgbs, op=dist.ReduceOp.MIN)
        med = statistics.median(times)
        res = {"n_total": n_tot, "value": round(n_tot / (med * 1e-3) / 1e6, 4), "ms_per_step": round(med, 4),
               "ms_min": round(min(times), 4), "ms_mean": round(statistics.mean(times), 4),
               "validation": {"pairs": int(bp.item()), "boundaries": boundary_bad, "multiset_hash_equal": hash_ok,
                              "steps": steps},
               "outcome": outc, "clocks": clk.summary(), "stages_rank0": stages,
               "gpu_launches": launches // max(steps, 1), "roofline": roof,
               "nvlink": {"bytes_to_peers_max_rank": int(to.item()),
                          "exchange_ms_rank0": round(xms, 4),
                          "achieved_gbs_min_rank": round(float(xgbs[0].item()), 1), "peak_gbs": 900.0,
                          "frac": round(float(xgbs[0].item()) / 900.0, 4),
                          "note": "string bytes + 8 B per string a rank sends to other ranks (peer stores into the "
                                  "destinations' NCCL windows) / the exchange kernel's time (profiled step); "
                                  "peak: NVLink 5 per direction per GPU"}}
        # e2e: pinned host block in, shard out, every step -- pipelined like
        # husky_sort_host_many: batch i+1's block goes in on a copy stream while
        # batch i is sorted, batch i's shard comes out on a third stream while
        # batch i+1 is sorted (two device input slots; each call's outputs are
        # fresh tensors, kept alive until their copy-out has finished)
        if want_e2e:
            hu = torch.empty(u.numel(), dtype=u.dtype).pin_memory()
            hu.copy_(u)
            ho = o.cpu().pin_memory()
            dus, dos = [torch.empty_like(u) for _ in range(2)], [torch.empty_like(o) for _ in range(2)]
            cap_n, cap_u = 2 * max(p.numel(), n_loc) + 1024, 2 * max(su.numel(), u.numel()) + 1024
            hp = torch.empty(cap_n, dtype=torch.int32).pin_memory()
            hsu = torch.empty(cap_u, dtype=u.dtype).pin_memory()
            hso = torch.empty(cap_n + 1, dtype=torch.int64).pin_memory()
            sh, sd = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
            K = args.e2e_steps
            h2d = hu.numel() * hu.element_size() + ho.numel() * 8

            def run_pipeline(k_batches):
                ev_in = [torch.cuda.Event() for _ in range(2)]
                ev_used = [None, None]  # the sort that last read input slot j
                live = []
                d2h_bytes = 0

                def issue_in(i):
                    j = i % 2
                    with torch.cuda.stream(sh):
                        if ev_used[j] is not None:
                            sh.wait_event(ev_used[j])
                        dus[j].copy_(hu, non_blocking=True)
                        dos[j].copy_(ho, non_blocking=True)
                        ev_in[j].record(sh)

                issue_in(0)
                for i in range(k_batches):
                    j = i % 2
                    if i + 1 < k_batches:
                        issue_in(i + 1)
                    stream.wait_event(ev_in[j])
                    ps, sus, sos, _ = h.sort_multi(comm, coder, dus[j], dos[j], base)
                    done = torch.cuda.Event()
                    done.record(stream)
                    ev_used[j] = done
                    with torch.cuda.stream(sd):
                        sd.wait_event(done)
                        k, ku = ps.numel(), sus.numel()
                        hp[:k].copy_(ps, non_blocking=True)
                        hsu[:ku].copy_(sus, non_blocking=True)
                        hso[:sos.numel()].copy_(sos, non_blocking=True)
                        for t in (ps, sus, sos):
                            t.record_stream(sd)
                    d2h_bytes = k * 4 + ku * sus.element_size() + sos.numel() * 8
                    live = [(ps, sus, sos)]
                torch.cuda.synchronize()
                del live
                return d2h_bytes

            run_pipeline(2)  # warm-up
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d2h = run_pipeline(K)
            ms = (time.perf_counter() - t0) * 1e3 / K
            et = torch.tensor([ms], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(et, op=dist.ReduceOp.MAX)
            res["e2e"] = {"value": round(n_tot / (float(et.item()) * 1e-3) / 1e6, 4), "unit": UNIT,
                          "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                          "ms_per_step": round(float(et.item()), 3),
                          "api": f"husky_sort_multi per rank, {K} steps as {K} pipelined batches: pinned host block "
                                 "-> device on a copy stream (two device input slots), sample sort, shard -> pinned "
                                 "host on a third stream (bytes of rank 0; time = max over ranks of the host wall "
                                 "clock around the K batches / K)"}
        return res

    main = one(name, n_total, args.steps, args.warmup, not args.no_e2e)
    n_loc = (rank + 1) * n_total // world - rank * n_total // world
    also = {}
    if not args.no_also and name == "C5":
        also["C4"] = one("C4", W.FULL_N["C4"], args.steps, args.warmup, False)
        also["C4"]["workload"] = DESCR["C4"]
    if rank == 0:
        line = {"metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "ms_min": main["ms_min"],
                "ms_mean": main["ms_mean"], "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u8", "data": "synthetic",
                "config": {"workload": DESCR[name], "n_total": n_total, "n_per_gpu": n_loc,
                           "parallelism": f"sample sort over {world} GPU(s), one dataset sharded by global index",
                           "timing": "per step: max over ranks of the CUDA-event time; median over steps",
                           "l2": "inputs > L2; a 256 MiB buffer is also written between timed steps"},
                "roofline": main["roofline"], "cpu_baseline": None, "e2e": main.get("e2e"),
                "gpu_launches": main["gpu_launches"],
                "clocks": main["clocks"], "validation": main["validation"], "nvlink": main["nvlink"],
                "stages": main["stages_rank0"],
                "outcome": main["outcome"], "also": also or None}
        print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    h.husky_comm_destroy(comm)  # releases the receive window (collective) before the NCCL comm
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2012_00866_b200 as h

    rank, world, local = dist_env()
    args.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    try:
        if world == 1 and not args.force_multi:
            return run_single(args, h, torch, dev)
        return run_sharded(args, h, torch, dev, rank, world)
    finally:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(DESCR))
    ap.add_argument("--n", type=int, default=0, help="strings in the dataset (default: the config's full size)")
    ap.add_argument("--cpu-sample", type=int, default=1 << 21)
    ap.add_argument("--ref-sample", type=int, default=1 << 21)
    # e2e batches per timed call: the pipeline's first H2D and last D2H are not
    # overlapped, so a few more batches than 3 show the steady state
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-also", action="store_true")
    ap.add_argument("--no-library-bar", action="store_true")
    ap.add_argument("--force-multi", action="store_true",
                    help="run the NCCL sample-sort path even on one GPU (validation)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
