#!/usr/bin/env python
"""Benchmark of the Huskysort hot path on B200 (BASELINE.json metric: strings
sorted/sec at 1/2/4/8 B200; radix/encode HBM GB/s vs peak).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C2] [--n N]

A step = one full husky_sort (encode -> onesweep radix -> run scan/check ->
fix-up -> gather) of one batch of synthetic strings through the C ABI, inputs
already resident in HBM.  N = 1 runs BASELINE.json configs[1] (C2: 1e7
English-like Zipf words); N > 1 (torchrun, one rank per GPU) runs the NCCL
sample sort with each rank holding its own 1e7-string block (weak scaling).
Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the
reference arm of this tier: there is no reference implementation, only the
paper) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
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
    "C5": "C5: len U[8,24] [0-9A-Za-z], 1% duplicates, first 10% pre-sorted, ASCII coder",
}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.25)
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
        mx = max(r[1] for r in rows)
        load = [r[0] for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows)}


def mean_prefix(w, K):
    L = w.offsets[1:] - w.offsets[:-1]
    return float(np.minimum(L, K).mean()), float(L.mean())


def cpu_baseline(name, n_sample):
    """The oracle as it stands (single-threaded C merge sort), on the host cores."""
    import oracle
    oracle.build()
    w = W.make(name, n_sample)
    # repeat the sort until about 10 s of CPU work (bounded: at most 8 calls)
    calls, dt = 0, 0.0
    while calls < 8 and (calls == 0 or dt < 10.0):
        t0 = time.perf_counter()
        oracle.sort(w.coder, w.units, w.offsets)
        dt += time.perf_counter() - t0
        calls += 1
    return {"value": round(n_sample * calls / dt / 1e6, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{name} generator, n={n_sample} strings, {calls} oracle_sort calls (top-down merge sort, "
                      f"1 thread), {dt:.2f} s wall in total"}


EXCHANGE = {1: "send buffers + ncclSend/ncclRecv",
            2: "gather stores straight into the peers' NCCL symmetric windows (NVLink), 4-byte all-reduce barrier"}


def make_config(args, n, coder, world):
    return {"workload": DESCR[args.config], "n_per_gpu": n, "coder": "ascii" if coder == 0 else "unicode",
            "outputs": "perm + sorted units + sorted offsets",
            "l2": "256 MiB buffer written between timed steps (outside the step events)",
            "parallelism": (f"sample sort over {world} GPU(s)" if world > 1 or getattr(args, "force_multi", False)
                            else "1 GPU")}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    n_sample = args.ref_sample
    w = W.make(args.config, n_sample)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.sort(w.coder, w.units, w.offsets)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    value = n_sample / t / 1e6
    sample = (f"{args.config} generator, n={n_sample} strings per step (bounded sample of the "
              f"{W.FULL_N[args.config]}-string workload), oracle_sort, 1 thread")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8" if w.coder == 0 else "u16", "data": "synthetic",
            "config": make_config(args, W.FULL_N[args.config] if not args.n else args.n, w.coder, 1),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2012_00866_b200 as h

    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    n = args.n or W.FULL_N[args.config]
    w = W.make(args.config, n, seed_offset=rank if world > 1 else 0)
    K = 9 if w.coder == 0 else 4
    p_bar, l_bar = mean_prefix(w, K)
    ub = w.unit_bytes
    units_np = w.units.view(np.int16) if ub == 2 else w.units
    d_units = torch.from_numpy(np.ascontiguousarray(units_np)).to(dev)
    d_off = torch.from_numpy(w.offsets).to(dev)
    total_units = w.units.size
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    if world == 1 and not args.force_multi:
        ws = torch.empty(h.husky_sort_workspace(w.coder, n, total_units), dtype=torch.uint8, device=dev)
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        su = torch.empty(total_units + 8, dtype=d_units.dtype, device=dev)
        so = torch.empty(n + 1, dtype=torch.int64, device=dev)

        def step():
            return h.husky_sort(w.coder, d_units, d_off, perm, su, so, ws)
    else:
        if world > 1:
            comm = h.multi.comm_from_process_group(device=dev)
        else:  # --force-multi on one GPU: the NCCL sample-sort path with a 1-rank communicator
            comm = h.husky_comm_create(0, 1, h.husky_comm_unique_id())
            h.multi._WORLD[comm.value] = 1
        gbase = rank * n

        def step():
            return h.sort_multi(comm, w.coder, d_units, d_off, gbase)[3]

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        outc = step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (outside the events).
    # Profiler mode 2: one event pair around the radix passes and one around the
    # encoder per step (the kernels' own stream), so the roofline durations are
    # measured live in the timed region at ~4 event records per step.
    h.husky_profile_reset()
    h.husky_profile_enable(2)
    l0 = h.husky_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            outc = step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = h.husky_launch_count() - l0
    h.husky_profile_enable(False)
    prof = h.husky_profile_read()
    # per-stage breakdown from separate steps with an event pair per launch
    # (informational: those per-launch records add ~0.1 ms to a step)
    h.husky_profile_reset()
    h.husky_profile_enable(1)
    n_bd = 3
    for i in range(n_bd):
        flush.fill_(i & 0xFF)
        step()
    torch.cuda.synchronize()
    h.husky_profile_enable(False)
    prof_bd = h.husky_profile_read()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    t_local = ms / args.steps
    if world > 1:
        t = torch.tensor([t_local], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t.item())
    else:
        t_step = t_local
    value = world * n / (t_step * 1e-3) / 1e6

    # ---- roofline of the dominant kernel (onesweep radix pass) and the encoder
    peak, peak_src = peaks()
    rp = prof["radix_pass"]
    # All 8 pass slots are launched (the pass plan is made on the device); the
    # ones beyond the plan exit at once and their time stays in the stage total.
    # Algorithmic bytes count the planned passes only.
    # main key-sort passes (refinement passes of A6 are not in the timed group)
    passes = int(outc.get("keys_partitioned", 0)) // n if isinstance(outc, dict) and n else 0
    radix_launches = passes * args.steps
    radix_bytes = 24 * n * radix_launches
    radix_gbs = radix_bytes / (rp["ms"] * 1e-3) / 1e9 if rp["ms"] else 0.0
    ep = prof["encode"]
    # encode: offsets 8 + prefix units + code 8 + packed payload 4 (n <= 2^28)
    enc_per = 8 + ub * p_bar + 8 + (4 if n <= (1 << 28) else 0)
    enc_bytes = n * args.steps * enc_per
    enc_gbs = enc_bytes / (ep["ms"] * 1e-3) / 1e9 if ep["ms"] else 0.0
    stages = {k: {"ms_per_step": round(v["ms"] / n_bd, 4), "launches_per_step": v["launches"] / n_bd}
              for k, v in prof_bd.items() if v["launches"]}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            td = json.load(open(tp)).get(args.config, {}).get("radix_pass")
            if td:
                traffic = int(td["bytes_per_key"] * n)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": "k_onesweep (A2 radix pass)",
                "achieved": round(radix_gbs, 1), "peak": peak, "unit": "GB/s",
                "frac": round(radix_gbs / peak, 4), "traffic": traffic,
                "bytes_alg_per_launch": int(radix_bytes / max(radix_launches, 1)),
                "ms_per_launch": round(rp["ms"] / max(radix_launches, 1), 5),
                "passes_per_sort": passes,
                "timing": "CUDA events around the pass group on the library's stream, every timed step",
                "alg_bytes_model": "24 B/key per pass (key 8 + payload 4, read + write; the first pass reads "
                                   "the packed index|len payload written by encode)",
                "peak_source": peak_src,
                "encode": {"achieved": round(enc_gbs, 1), "frac": round(enc_gbs / peak, 4),
                           "ms_per_launch": round(ep["ms"] / args.steps, 5),
                           "alg_bytes_model": f"{enc_per:.2f} B/string: offset 8 + code 8 + payload 4 + {ub} B x "
                                              f"mean min(len,{K}) = {p_bar:.2f} units"}}

    # ---- end to end through the C ABI with HOST buffers (H2D/D2H inside the timed region)
    e2e = None
    if world == 1 and not args.force_multi:
        hu = torch.from_numpy(np.ascontiguousarray(units_np)).pin_memory()
        ho = torch.from_numpy(w.offsets).pin_memory()
        hp = torch.empty(n, dtype=torch.int32).pin_memory()
        hsu = torch.empty(total_units + 8, dtype=d_units.dtype).pin_memory()
        hso = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        ws = None  # free the device workspace before the host-API workspace
        torch.cuda.empty_cache()
        hws = torch.empty(h.husky_sort_host_workspace(w.coder, n, total_units), dtype=torch.uint8, device=dev)
        for _ in range(max(1, args.warmup)):
            h.husky_sort_host(w.coder, hu, ho, hp, hsu, hso, hws)
        torch.cuda.synchronize()
        e_ms = 0.0
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            h.husky_sort_host(w.coder, hu, ho, hp, hsu, hso, hws)
            b.record(stream)
            torch.cuda.synchronize()
            e_ms += a.elapsed_time(b)
        e_ms /= args.steps
        single = {"value": round(n / (e_ms * 1e-3) / 1e6, 4), "ms_per_step": round(e_ms, 3),
                  "api": "husky_sort_host, one call per step (pinned host buffers)"}
        # pipelined: the K steps as K batches of husky_sort_host_many (2 device
        # buffer slots, one stream each for H2D copies, kernels and D2H copies),
        # so one step's copies overlap another's kernels and the full-duplex
        # PCIe carries H2D and D2H at once
        depth = int(os.environ.get("HUSKY_E2E_DEPTH", "2"))
        hws = None
        torch.cuda.empty_cache()
        mws = torch.empty(h.husky_sort_host_many_workspace(w.coder, n, total_units, depth), dtype=torch.uint8,
                          device=dev)
        outs = [(torch.empty(n, dtype=torch.int32).pin_memory(),
                 torch.empty(total_units + 8, dtype=d_units.dtype).pin_memory(),
                 torch.empty(n + 1, dtype=torch.int64).pin_memory()) for _ in range(depth)]
        batches = [(hu, ho, outs[b % depth][0], outs[b % depth][1], outs[b % depth][2]) for b in range(args.steps)]
        h.husky_sort_host_many(w.coder, batches[:depth], mws, depth)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.husky_sort_host_many(w.coder, batches, mws, depth)
        torch.cuda.synchronize()
        p_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        e2e = {"value": round(n / (p_ms * 1e-3) / 1e6, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(total_units * ub + (n + 1) * 8),
               "d2h_bytes_per_step": int(n * 4 + total_units * ub + (n + 1) * 8),
               "ms_per_step": round(p_ms, 3),
               "api": f"husky_sort_host_many: {args.steps} steps as {args.steps} pipelined batches, {depth} "
                      "device slots, H2D / kernels / D2H on three streams (pinned host buffers), host wall clock "
                      "around the call",
               "single_call": single}
    elif world > 1 or args.force_multi:
        # sharded: every step copies the rank's input block from pinned host
        # memory, runs the sample sort, and reads its output shard back; time =
        # max over ranks of the CUDA-event time on the current stream
        hu = torch.from_numpy(np.ascontiguousarray(units_np)).pin_memory()
        ho = torch.from_numpy(w.offsets).pin_memory()
        du = torch.empty_like(d_units)
        do = torch.empty_like(d_off)
        # shard sizes vary with the splitters: pinned output buffers with slack
        p0, su0, so0, _ = h.sort_multi(comm, w.coder, d_units, d_off, gbase)
        cap_n, cap_u = 2 * max(p0.numel(), n) + 1024, 2 * max(su0.numel(), total_units) + 1024
        hp = torch.empty(cap_n, dtype=torch.int32).pin_memory()
        hsu = torch.empty(cap_u, dtype=d_units.dtype).pin_memory()
        hso = torch.empty(cap_n + 1, dtype=torch.int64).pin_memory()
        e_ms, h2d, d2h = 0.0, 0, 0
        for i in range(args.steps + max(1, args.warmup)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a.record(stream)
            du.copy_(hu, non_blocking=True)
            do.copy_(ho, non_blocking=True)
            perm_s, su_s, so_s, _ = h.sort_multi(comm, w.coder, du, do, gbase)
            k, ku = perm_s.numel(), su_s.numel()
            hp[:k].copy_(perm_s, non_blocking=True)
            hsu[:ku].copy_(su_s, non_blocking=True)
            hso[:so_s.numel()].copy_(so_s, non_blocking=True)
            b.record(stream)
            torch.cuda.synchronize()
            if i < max(1, args.warmup):
                continue  # warm-up (first use of these buffers by the exchange)
            e_ms += a.elapsed_time(b)
            h2d = hu.numel() * hu.element_size() + ho.numel() * 8
            d2h = k * 4 + ku * su_s.element_size() + so_s.numel() * 8
        e_ms /= args.steps
        if world > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": round(world * n / (e_ms * 1e-3) / 1e6, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e_ms, 3),
               "api": "husky_sort_multi per rank: pinned host block -> device, sample sort, shard -> pinned host "
                      "(bytes of rank 0; time = max over ranks)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, min(n, args.cpu_sample))

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(t_step, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u8" if ub == 1 else "u16",
                "data": "synthetic",
                "config": dict(make_config(args, n, w.coder, world),
                               **({"exchange": EXCHANGE.get(outc.get("exchange", 0), "?")}
                                  if isinstance(outc, dict) and outc.get("exchange") else {})),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk.summary(), "stages": stages, "outcome": outc}
        print(json.dumps(line), flush=True)
    if world > 1 or args.force_multi:
        torch.cuda.synchronize()
        h.husky_comm_destroy(comm)  # releases the receive window (collective) before the NCCL comm
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(DESCR))
    ap.add_argument("--n", type=int, default=0, help="strings per GPU (default: the config's full size)")
    ap.add_argument("--cpu-sample", type=int, default=10_000_000)
    ap.add_argument("--ref-sample", type=int, default=4_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
