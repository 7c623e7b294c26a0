#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric):
"3D DRT Gvoxel/s (N=256, 12 dodecants) and achieved HBM GB/s vs B200 peak".

Workload (BASELINE config 3): one N=256 uint8 cube, 30% of voxels non-zero
U{1..255} (synth.config_input(3)), all 12 dodecants, int32 output
[12][256][256][768] (2.416 GB) in the stacked layout.

One step = one full drt3d_planes call (every pass of every dodecant) with the
cube already resident in HBM.  W warm-up steps, then exactly K timed steps
bracketed by barrier + synchronize; each step is timed with CUDA events on the
launching stream; between steps a 512 MB buffer is rewritten to flush the
126 MB L2 (outside the per-step events).  Multi-GPU: one process per GPU, each
rank transforms its own cube (independent problems, weak scaling, no
data-path collective); time = max over ranks.

Extra keys: roofline of the dominant kernel (final pass), cpu_baseline (the
oracle's Alg. 1 on host cores), e2e through the host-buffer C entry point,
clocks sampled by nvidia-smi during the timed region.

`--impl reference` times the CPU oracle (this tier's reference arm) on the
same config, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 256
MASK = 0xFFF
K_DOD = 12
METRIC = "3D DRT Gvoxel/s (N=256, 12 dodecants) and achieved HBM GB/s vs B200 peak"
WORKLOAD = "cfg3_drt_n256_u8_sparse30_12dod"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks
_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
            0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index: int):
        self.index, self.samples, self.proc, self.thread = index, [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [t.strip() for t in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        mask = 0
        for _, _, r in self.samples:
            mask |= r
        reasons = [n for b, n in _REASONS.items() if mask & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ multi-rank plumbing
def max_over_ranks(x: float, world: int, device=None) -> float:
    """Max of a per-rank scalar over all ranks (timing rule: max over ranks)."""
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_gvoxels(units_per_rank: float, world: int, ms_per_step: float) -> float:
    """Whole-job throughput: every rank transforms its own cube (weak scaling)."""
    return world * units_per_rank / (ms_per_step * 1e-3) / 1e9


# ------------------------------------------------------------ CPU oracle arm
def _oracle_dodecant(k: int) -> float:
    import numpy as np
    import oracle
    import synth
    from oracle import tables
    f = synth.config_input(3)[0]
    g = oracle.orient(f, tables.DRT_HEMISPHERE[k])
    t = time.perf_counter()
    out = oracle.drt_alg1(g)
    dt = time.perf_counter() - t
    assert out.shape == (N, N, 3 * N)
    return dt


def cpu_oracle_sample(workers: int) -> dict:
    """Alg. 1 (oracle/oracle.c, int64, single-threaded per process) on `workers`
    dodecants of the cfg3 cube in parallel processes (the paper's dodecant
    parallelism).  Gvoxel/s = (workers/12) * N^3 / wall."""
    import concurrent.futures as cf
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    if workers == 1:
        per = [_oracle_dodecant(0)]
    else:
        with cf.ProcessPoolExecutor(workers) as ex:
            per = list(ex.map(_oracle_dodecant, range(workers)))
    wall = time.perf_counter() - t0
    return {"wall_s": wall, "per_dodecant_s": per, "value": (workers / K_DOD) * N ** 3 / wall / 1e9}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    workers = max(1, min(K_DOD, cores))
    for _ in range(args.warmup):
        if args.warmup_reference:
            cpu_oracle_sample(workers)
    vals, walls = [], []
    for _ in range(args.steps):
        r = cpu_oracle_sample(workers)
        vals.append(r["value"])
        walls.append(r["wall_s"])
    value = args.steps * (workers / K_DOD) * N ** 3 / sum(walls) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gvoxel/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / len(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "N": N, "dodecants": K_DOD, "in_dtype": "u8", "out_dtype": "int64"},
        "cpu_baseline": {"value": value, "unit": "Gvoxel/s", "cores": workers, "kind": "oracle",
                         "sample": f"Alg. 1 (oracle/oracle.c) on {workers} of 12 dodecants of the cfg3 cube per step, "
                                   f"one process per dodecant"},
        "e2e": {"value": value, "unit": "Gvoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU arm
def run_ours(args):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2501_13664_b200 as d3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    cube_h = synth.config_input(3)                                # [1][N][N][N] uint8 (each rank: own replica)
    cube = torch.from_numpy(cube_h).to(dev)
    out = torch.empty((1, K_DOD, N, N, 3 * N), dtype=torch.int32, device=dev)
    opts = d3.make_opts(batch=1, in_dtype=d3.DRT3D_U8, out_dtype=d3.DRT3D_I32)
    ws_bytes = d3.drt3d_planes_workspace_size(N, MASK, opts)
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    # per-launch events (instrumentation through the C ABI)
    max_ev = 64
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * max_ev)]
    for e in evs:                      # torch creates events lazily: force creation
        e.record(stream)
    torch.cuda.synchronize()
    ev_arr = (ctypes.c_void_p * (2 * max_ev))(*[e.cuda_event for e in evs])
    n_launch = ctypes.c_int(0)
    kinds = (ctypes.c_int * max_ev)()
    opts.events = ctypes.cast(ev_arr, ctypes.c_void_p)
    opts.max_events = max_ev
    opts.launches = ctypes.pointer(n_launch)
    opts.launch_kind = ctypes.cast(kinds, ctypes.POINTER(ctypes.c_int))

    def step():
        s = d3.drt3d_planes(cube.data_ptr(), N, MASK, out.data_ptr(), opts, ws.data_ptr(), ws_bytes,
                            stream.cuda_stream)
        if s != d3.DRT3D_OK:
            raise RuntimeError(d3.status_string(s))

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kind_ms = {0: [], 1: [], 2: []}
    launches = 0
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    for i in range(args.steps):
        flush.zero_()
        starts[i].record(stream)
        step()
        stops[i].record(stream)
        stream.synchronize()           # read this step's per-launch events before they are re-recorded
        launches += n_launch.value
        for j in range(min(n_launch.value, max_ev)):
            if kinds[j] in kind_ms:
                kind_ms[kinds[j]].append(evs[2 * j].elapsed_time(evs[2 * j + 1]))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, stops)]
    tot_ms = max_over_ranks(sum(step_ms), world, dev)
    ms_per_step = tot_ms / args.steps
    value = whole_job_gvoxels(N ** 3, world, ms_per_step)          # Gvoxel/s, whole job

    peak, peak_kind = _peaks()
    # algorithmic bytes: whole call = cube read once + output written once
    call_bytes = N ** 3 * 1 + K_DOD * N * N * 3 * N * 4
    # dominant kernel = final pass; per dodecant it reads the stage-4 partial transform on its
    # support (N^2 rows x (N+30) u16) and writes N^2 x 3N int32.  One launch covers all the
    # dodecants of a chunk (12 at N=256: DESIGN.md §5), so the bytes per launch scale with that.
    final_launches_per_step = max(1, len(kind_ms[2]) // max(1, args.steps))
    dod_per_final_launch = K_DOD / final_launches_per_step
    final_bytes = int(dod_per_final_launch * (N * N * (N + 30) * 2 + N * N * 3 * N * 4))
    fin_ms = statistics.mean(kind_ms[2]) if kind_ms[2] else float("nan")
    first_ms = statistics.mean(kind_ms[0]) if kind_ms[0] else float("nan")
    achieved = final_bytes / (fin_ms * 1e-3) / 1e9
    # dram__bytes_read.sum + dram__bytes_write.sum of the final pass from the committed ncu --set full
    # capture (profiles/ncu_traffic.json, written by tools/ncu_traffic.py from that report)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        traffic, traffic_src = tj.get("final_pass_dram_bytes_per_launch"), tj.get("source")
    share = sum(kind_ms[2]) / max(1e-9, sum(kind_ms[0]) + sum(kind_ms[1]) + sum(kind_ms[2]))
    # context: the incompressible write-only HBM ceiling measured on this GPU type (the final pass is
    # ~83% writes), profiles/r2_hbm_ceilings.json (tools/hbm_write_probe.py)
    wceil = None
    cpath = os.path.join(ROOT, "profiles", "r2_hbm_ceilings.json")
    if os.path.exists(cpath):
        with open(cpath) as fh:
            wceil = json.load(fh).get("write_only_ceiling_gbs")

    # e2e through the host-buffer C entry point (pinned host cube + output)
    e2e = None
    if args.e2e_steps > 0:
        hcube = torch.from_numpy(cube_h).pin_memory()
        hout = torch.empty(out.shape, dtype=torch.int32, pin_memory=True)
        dcube = torch.empty_like(cube)
        o2 = d3.make_opts(batch=1, in_dtype=d3.DRT3D_U8, out_dtype=d3.DRT3D_I32)

        def e2e_step():
            s = d3.drt3d_planes_host(hcube.data_ptr(), N, MASK, hout.data_ptr(), o2, dcube.data_ptr(),
                                     out.data_ptr(), ws.data_ptr(), ws_bytes, stream.cuda_stream)
            if s != d3.DRT3D_OK:
                raise RuntimeError(d3.status_string(s))
        e2e_step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = max_over_ranks(a.elapsed_time(b) / args.e2e_steps, world, dev)
        # spot-check that the e2e result is the device result
        assert bool((hout[0, 0, 0, 0].to(dev) == out[0, 0, 0, 0]).all())
        e2e = {"value": whole_job_gvoxels(N ** 3, world, e_ms), "unit": "Gvoxel/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(cube.numel()), "d2h_bytes_per_step": int(out.numel() * 4)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_oracle_sample(1)
        cpu = {"value": r["value"], "unit": "Gvoxel/s", "cores": 1, "kind": "oracle",
               "sample": "Alg. 1 (oracle/oracle.c, int64) on dodecant 0 of the cfg3 cube, 1 thread; "
                         "Gvoxel/s = N^3 / (12 x one-dodecant time)", "seconds": r["wall_s"]}

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gvoxel/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "N": N, "dodecants": K_DOD, "in_dtype": "u8", "out_dtype": "i32",
                       "layout": "stacked [12][N][N][3N]", "table": "hemisphere",
                       "l2": "512 MB flush write between timed steps (outside per-step events)",
                       "parallelism": f"replicas x{world} (one cube per GPU)"},
            "gplanes_per_s": world * K_DOD * N * N * (2 * N - 1) / (ms_per_step * 1e-3) / 1e9,
            "call_hbm_gbs_algorithmic": call_bytes / (ms_per_step * 1e-3) / 1e9,
            "call_frac_of_peak": call_bytes / (ms_per_step * 1e-3) / 1e9 / peak,
            "roofline": {"kernel": "drt_pass_kernel<K=4> final pass", "bound": "hbm", "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": final_bytes, "dodecants_per_launch": dod_per_final_launch,
                         "launch_ms": fin_ms, "first_pass_ms": first_ms, "share_of_step": share,
                         "write_ceiling_gbs": wceil, "frac_of_write_ceiling": achieved / wceil if wceil else None},
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------ CPU oracle per BASELINE config
# (the oracle beside every configuration; part of the reference arm, the
# only place besides the cpu_baseline leg where bench.py executes oracle/)
_CUBES = {}


def _oracle_job(args):
    import oracle
    import synth
    from oracle import tables
    cfg, kind, b, k = args
    if cfg not in _CUBES:                      # once per process: the inputs are large to regenerate
        _CUBES[cfg] = synth.config_input(cfg)
    cube = _CUBES[cfg][b]
    if kind == "drt":
        oracle.drt_alg1(oracle.orient(cube, tables.DRT_HEMISPHERE[k]))
    else:
        oracle.djt_alg3(oracle.orient(cube, tables.table(tables.TABLE_HEMISPHERE, "djt")[k]))
    return 0


def _timed(jobs, workers, reps):
    from concurrent.futures import ProcessPoolExecutor
    best = 1e30
    for r in range(reps + 1):                  # one warm-up, then best of reps
        t0 = time.perf_counter()
        if workers == 1:
            for j in jobs:
                _oracle_job(j)
        else:
            with ProcessPoolExecutor(workers) as ex:
                list(ex.map(_oracle_job, jobs))
        dt = time.perf_counter() - t0
        if r > 0:
            best = min(best, dt)
    return best


def run_reference_configs(args):
    """T=1 (one process) and T=all (one process per dodecant or cube) oracle wall time for each
    BASELINE config on this host; config 3 times single dodecants (about 11 s each) and scales by
    the dodecant count.  One JSON line per config."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cores = os.cpu_count() or 1
    specs = {1: ("drt", 1, [0]), 2: ("drt", 1, range(12)), 4: ("djt", 1, [0]), 5: ("drt", 256, range(12))}
    for cfg, (kind, nb, ks) in specs.items():
        jobs = [(cfg, kind, b, k) for b in range(nb) for k in ks]
        reps = 1 if cfg == 5 else 3
        t1 = _timed(jobs, 1, reps)
        ta = _timed(jobs, min(cores, len(jobs)), reps)
        print(json.dumps({"impl": "reference", "config": cfg, "oracle_T1_ms": 1e3 * t1, "oracle_Tall_ms": 1e3 * ta,
                          "cores": min(cores, len(jobs))}), flush=True)
    t1 = _timed([(3, "drt", 0, 0)], 1, 1)
    w = min(cores, 12)
    ta = _timed([(3, "drt", 0, k) for k in range(12)], w, 1)
    print(json.dumps({"impl": "reference", "config": 3, "oracle_T1_ms": 12e3 * t1, "oracle_T1_note": "12 x one dodecant",
                      "oracle_Tall_ms": 1e3 * ta, "cores": w}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--warmup-reference", action="store_true",
                    help="also run the (slow) oracle during warm-up steps of --impl reference")
    ap.add_argument("--configs", action="store_true",
                    help="with --impl reference: time the oracle on every BASELINE config (BASELINE.md section 4)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference" and args.configs:
        run_reference_configs(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
