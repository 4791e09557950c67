#!/usr/bin/env python
"""Benchmark: BASELINE.json configs[1] (C2) — AoS->SoA conversion with
binary16 storage of position/velocity, fused into drift, 16M particles.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one pass of the hot path over the whole 16M-particle population:
the default 88-B AoS (f64 x, f32 v, ...) in HBM -> k_gather_xv_staged (each
CTA's records staged in shared memory by one TMA bulk copy, RNE narrowing to
binary16, drift x += v*dt in binary64) ->
SoA binary16 {x', v}.  Under torchrun every rank runs its own 16M particles
(weak scaling: particles shard with no data-path collective); timing is the
max over ranks.  `e2e` is the same step through the C ABI with HOST buffers
(pinned AoS in, SoA out, chunked H2D/compute/D2H pipeline inside the timed
region).  `--impl reference` times the unmodified reference (oracle/_ref) on
this host's cores for the same composition.

`--gpus N` (N > 1) without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, NCCL).  The default line also
carries the other BASELINE configs and the paper's measurements as extra
keys (skip them with --no-extras): configs.c1 / c3 / c4 (each with its own
roofline and cpu_baseline), sharded_c5 (the 128M cell-sharded timestep at
every N, strong scaling, per-phase ms), soa_vs_aos, transform and timestep.
"""
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

METRIC = "particle updates/s & HBM GB/s vs peak per kernel; GPU vs CPU AoS→SoA speedup"
UNIT = "particle updates/s"
N_DEFAULT = 1 << 24
REC_BYTES = 88
ALG_BYTES = 48  # R x(f64) 24 + v(f32) 12, W SoA x' 6 + v 6


def config(n, world, prec_name):
    return {"workload": "C2 (BASELINE configs[1]): AoS->SoA + %s storage of x,v fused into drift" % prec_name,
            "particles_per_gpu": n, "record_bytes": REC_BYTES, "schema": "reference default (f64 x3, i64, f32 ...)",
            "dst": "SoA %s {x', v}" % prec_name, "dt": 1e-3, "arith": "binary64, separately rounded (bit-exact)",
            "l2": "inputs 1.48 GB/GPU > 126 MB L2; no flush needed",
            "parallelism": "replicas" if world == 1 else "dp%d (particles sharded, no collective)" % world}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic_from_profiles(kernel_key):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel_key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the GPU is busy."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.samples, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def cpu_reference_rate(n_per_thread, threads, prec, seed=42):
    """The unmodified reference (oracle/_ref) C2 composition on host cores."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.RefLib.available():
        raise RuntimeError("oracle/_ref/libref_driver.so missing (run `make -C oracle`)")
    R = O.RefLib()
    T = 16
    secs = R.time_c2(n_per_thread, threads, T, seed)
    if secs <= 0:
        raise RuntimeError(R.L.ref_last_error().decode())
    return n_per_thread * threads / secs, secs


def cpu_c1_rate(n, threads, dt=1e-3, kernels=("kick", "drift")):
    """C1 on the unmodified reference itself (oracle/_ref): kick then drift in
    place on the default AoS (run_kernel_chunked, 64-particle buffers, `threads`
    host threads), the full 1M-particle workload."""
    import time
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.RefLib.available():
        raise RuntimeError("oracle/_ref/libref_driver.so missing (run `make -C oracle`)")
    R = O.RefLib()
    h = R.from_ics(n, 42, 0, "", None, 43, dt)
    R.run_kernel(h, kernels[0], 64, dt, threads=threads)  # warm-up: pages touched, threads spawned once
    t0 = time.perf_counter()
    for k in kernels:
        R.run_kernel(h, k, 64, dt, threads=threads)
    secs = time.perf_counter() - t0
    R.free(h)
    return n / secs, secs


def cpu_c3_port_rate(n_total, sample=1 << 16, seed=5):
    """C3's cell-linked density on the CPU: the oracle's C restatement
    (oracle/soa_oracle.c or_density_cells, one core) on a sub-box holding
    `sample` particles at C3's number density and smoothing length."""
    import time
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2512_05516_b200.sharded import grid_for
    h, _, _ = grid_for(n_total)
    side = (sample / n_total) ** (1.0 / 3.0)
    ncell = max(1, int(side / (2 * h)))
    rng = np.random.default_rng(seed)
    x = rng.random((sample, 3)) * side
    m = np.full(sample, 1.0 / n_total)
    hh = np.full(sample, h)
    t0 = time.perf_counter()
    O.density_cells(x.reshape(-1), m, hh, 0.0, side, side / ncell)
    secs = time.perf_counter() - t0
    return sample / secs, secs


def cpu_reference_kernels_rate(n, kernels, threads, T=32, layout="soa", seed=42):
    """The unmodified reference's own kernels (run_kernel_chunked, 64-particle
    buffers, binary64) on `threads` host threads over an n-particle population
    stored at T (x kept f64) and unpacked to `layout`: particles per second of
    the whole kernel list (e.g. density,force,kick,drift = one timestep)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.RefLib.available():
        raise RuntimeError("oracle/_ref/libref_driver.so missing (run `make -C oracle`)")
    R = O.RefLib()
    h = R.from_ics(n, seed, T, "x", None, 43, 1e-3)
    u = R.op(h, "unpack")
    buf = R.op(u, "aos_to_soa") if layout == "soa" else u
    R.run_kernel(buf, kernels[0], 64, 1e-3, threads=threads)  # warm-up: pages touched
    t0 = time.perf_counter()
    for k in kernels:
        R.run_kernel(buf, k, 64, 1e-3, threads=threads)
    secs = time.perf_counter() - t0
    R.free(*([h, u, buf] if buf is not u else [h, u]))
    return n / secs, secs


def _bench_kernels_csv(lib_path, particles, threads):
    """Run a library's sf_run_bench_kernels (bench.cpp:269-316 semantics)."""
    import ctypes as C
    L = C.CDLL(lib_path)
    L.sf_config_create.argtypes = [C.POINTER(C.c_void_p)]
    L.sf_config_set_int.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
    L.sf_config_set_string.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
    L.sf_run_bench_kernels.argtypes = [C.c_void_p, C.POINTER(C.c_char_p)]
    L.sf_config_destroy.argtypes = [C.c_void_p]
    L.sf_last_error.restype = C.c_char_p
    cfg = C.c_void_p()
    L.sf_config_create(C.byref(cfg))
    L.sf_config_set_int(cfg, b"particles", particles)
    L.sf_config_set_int(cfg, b"threads", threads)
    L.sf_config_set_string(cfg, b"kernels", b"kick,drift,density")
    L.sf_config_set_string(cfg, b"precision", b"64,32,16")
    out = C.c_char_p()
    st = L.sf_run_bench_kernels(cfg, C.byref(out))
    text = out.value.decode() if out.value else ""
    L.sf_config_destroy(cfg)
    if st != 0:
        raise RuntimeError(L.sf_last_error().decode())
    rows = [l.split(",") for l in text.splitlines() if l and not l.startswith("#")]
    head = rows[0]
    return [dict(zip(head, r)) for r in rows[1:]]


def kernels_table(particles):
    """Reference CPU (all host cores) vs this GPU library, per kernel x layout x
    precision, both through their own sf_run_bench_kernels on the same config:
    particle updates/s and the checksum agreement (north_star: AoS and SoA, each
    precision mode)."""
    threads = os.cpu_count() or 1
    ref = _bench_kernels_csv(os.path.join(ROOT, "oracle", "_ref", "libsoaforge_ref.so"), particles, threads)
    from paper_2512_05516_b200 import _lib
    gpu = _bench_kernels_csv(_lib.LIB_PATH, particles, threads)
    table = {}
    for r, g in zip(ref, gpu):
        key = "%s/%s/T%s" % (r["kernel"], r["layout"], r["precision"])
        cs, gs = float(r["compute_s"]), float(g["compute_s"])
        table[key] = {"cpu_updates_per_s": particles / cs if cs > 0 else None,
                      "gpu_updates_per_s": particles / gs if gs > 0 else None,
                      "checksum_equal": r["checksum"] == g["checksum"]}
    return {"particles": particles, "cpu_threads": threads, "rows": table,
            "note": "density = 64-particle buffer mode (reference semantics, binary64); GPU time excludes transfers; "
                    "at this size (the reference bench command's own scale, ~10 s of CPU) the GPU kick/drift rows are "
                    "launch-bound: soa_vs_aos holds the 16M-particle layout comparison"}


def dist_init():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # SFB_BENCH_ONE_DEVICE=1 (tests only): every rank on cuda:0 over gloo, to exercise the
        # multi-rank logic on a one-GPU box; production runs are one NCCL rank per GPU
        if os.environ.get("SFB_BENCH_ONE_DEVICE") == "1":
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
            return world, rank, 0
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def reference_arm(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n_pt = args.ref_sample // threads
    for _ in range(args.warmup):
        cpu_reference_rate(max(n_pt // 8, 128), threads, args.prec)
    times = []
    for _ in range(args.steps):
        rate, secs = cpu_reference_rate(n_pt, threads, args.prec)
        times.append(secs)
    total = n_pt * threads
    value = total * len(times) / sum(times)
    sample = "%d particles/step (%d per thread x %d threads) of the C2 workload; reference ops: " \
             "load_state->store_state(T16)->unpack->narrow(drift)->aos_to_soa->run_kernel_chunked(drift)" % (
                 total, n_pt, threads)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference random_initial_conditions, seed 42+thread)",
            "config": dict(config(N_DEFAULT, world, "binary16"), reference_sample_particles_per_step=total),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def b200_arm(args):
    import torch
    from paper_2512_05516_b200 import api

    world, rank, local = dist_init()
    dist = None
    if world > 1:
        import torch.distributed as dist
    n = args.n
    prec = api.SF_PREC_BF16 if args.prec == "bf16" else 16
    prec_name = "bf16" if args.prec == "bf16" else "binary16"
    P = api.Schema.default()
    aos_v = api.View(P, n, "aos")
    dst_v = api.View(P, n, "soa", "drift", prec)

    # synthetic population generated on the device (seeded per rank)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    src = api.PackedBuffer.empty(aos_v)
    rec = src.data[: aos_v.nbytes].view(n, REC_BYTES)
    step = 1 << 22
    for b in range(0, n, step):
        e = min(n, b + step)
        m = e - b
        f = torch.rand(m, 17, device="cuda", generator=g)
        rec[b:e, 0:24] = f[:, 0:3].double().contiguous().view(torch.uint8).view(m, 24)
        rec[b:e, 24:32] = torch.arange(b, e, device="cuda", dtype=torch.int64).view(torch.uint8).view(m, 8)
        f[:, 3:6] = f[:, 3:6] * 2 - 1  # v ~ U(-1, 1)
        rec[b:e, 32:88] = f[:, 3:17].contiguous().view(torch.uint8).view(m, 56)
    out = api.PackedBuffer.empty(dst_v)
    stream = torch.cuda.current_stream()

    def step_fn():
        api.gather_kernel(src, dst_v, "drift", 1e-3, api.SF_MATH_FP64_EXACT, out=out)

    def barrier():
        if dist is not None:
            dist.barrier()

    # warm-up (W) plus a ~0.5 s untimed soak so the clock sampler sees load
    for _ in range(max(args.warmup, 3)):
        step_fn()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    t_end = time.time() + 0.5
    while time.time() < t_end:
        for _ in range(20):
            step_fn()
        torch.cuda.synchronize()

    launches0 = api.launch_count()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step_fn()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    launches = api.launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = n * world / (ms_max * 1e-3)

    peak, peak_kind = peaks()
    achieved = ALG_BYTES * n / (ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_kind": peak_kind, "kernel": "k_gather_xv_staged (CTA records staged by TMA, fused gather+drift, %s)" % prec_name,
                "algorithmic_bytes_per_particle": ALG_BYTES,
                "traffic": traffic_from_profiles("gather_drift_%s" % args.prec)}
    if roofline["traffic"]:  # the DRAM bytes ncu measured per launch, over the same launch time
        roofline["dram_achieved"] = roofline["traffic"] / (ms * 1e-3) / 1e9
        roofline["dram_frac"] = roofline["dram_achieved"] / peak
        roofline["note"] = ("frac counts the 48 algorithmic B/particle; the 88-B AoS record crosses HBM whole "
                            "(DRAM fetch granularity >= 64 B, profiles/r01_sector_probe.md), so frac <= 0.48 "
                            "by format; dram_frac is the measured-bytes fraction of the copy peak")

    # SURVEY §8d C2 scatter-back row: the drifted SoA x' (binary16) widened exactly into the f64 x lanes of the
    # AoS records, every other byte untouched (widen_merge of the drift write set; 30 B/particle algorithmic)
    scatter = None
    if world == 1:
        tgt = api.PackedBuffer.empty(aos_v)  # a copy: the source AoS stays as generated for the e2e check
        tgt.data.copy_(src.data)
        for _ in range(3):
            api.widen_merge(out, tgt, "drift")
        torch.cuda.synchronize()
        sa, sb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(args.steps // 2, 10)
        sa.record(stream)
        for _ in range(reps):
            api.widen_merge(out, tgt, "drift")
        sb.record(stream)
        sb.synchronize()
        s_ms = sa.elapsed_time(sb) / reps
        scatter = {"ms": s_ms, "value": n / (s_ms * 1e-3), "algorithmic_bytes_per_particle": 30,
                   "achieved_GBps": 30 * n / (s_ms * 1e-3) / 1e9, "frac": 30 * n / (s_ms * 1e-3) / 1e9 / peak,
                   "kernel": "k_scatter_tile (records staged by one TMA bulk copy, binary16 x widened into the f64 "
                             "x lanes in shared memory, 256-bit write-back of the chunks holding x)",
                   "note": "the 24-B x lanes of an 88-B record straddle 32-B sectors and DRAM fetches >= 64 B, "
                           "so the whole record is read and 1-2 whole chunks written per record"}
        del tgt

    # end to end through the C ABI: pinned host AoS in, host SoA out
    e2e = None
    if not args.no_e2e:
        hb = api.HostBuffer(aos_v.nbytes, 0)
        hb_np = hb.numpy()
        torch.cuda.synchronize()
        chunk_b = 1 << 22
        for b in range(0, aos_v.nbytes, chunk_b * REC_BYTES):
            e = min(aos_v.nbytes, b + chunk_b * REC_BYTES)
            hb_np[b:e] = src.data[b:e].cpu().numpy()
        hs = api.HostBuffer(dst_v.nbytes, 0)
        for _ in range(max(1, min(args.warmup, 2))):
            api.run_host(aos_v, hb, dst_v, "drift", 1e-3, chunk=args.chunk, soa_out=hs, mode=2)
        barrier()
        secs = []
        for _ in range(args.e2e_steps):
            m = api.run_host(aos_v, hb, dst_v, "drift", 1e-3, chunk=args.chunk, soa_out=hs, mode=2)
            secs.append(m["seconds"])
        s_t = torch.tensor([sum(secs) / len(secs)], device="cuda", dtype=torch.float64)
        if dist is not None:
            dist.all_reduce(s_t, op=dist.ReduceOp.MAX)
        # parity of the e2e result with the device-resident result
        got = torch.from_numpy(hs.numpy()[: dst_v.nbytes].copy()).cuda()
        ok = bool(torch.equal(got, out.data[: dst_v.nbytes]))
        e2e = {"value": n * world / float(s_t.item()), "unit": UNIT, "h2d_bytes_per_step": m["h2d_bytes"] * world,
               "d2h_bytes_per_step": m["d2h_bytes"] * world, "chunk_particles": args.chunk, "matches_device_result": ok,
               "path": "sf_b200_run_host(mode 2): pinned AoS, whole records H2D || k_gather_xv_staged (fused drift) || "
                       "D2H SoA, 3-stream chunk pipeline"}
        hb.free()
        hs.free()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            n_pt = max(args.ref_sample // 4 // threads, 1024)
            rate, secs = cpu_reference_rate(n_pt, threads, args.prec)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": "%d particles (%d/thread) of C2 through the unmodified reference ops, %.2f s" % (
                       n_pt * threads, n_pt, secs)}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "unavailable: %s" % ex}
        try:
            cpu["per_mode"] = kernels_table(args.table_particles)
        except Exception as ex:
            cpu["per_mode"] = {"unavailable": str(ex)}

    extras = {}
    if not args.no_extras:
        del out, src
        torch.cuda.empty_cache()
        extras = run_extras(args, world, rank, peak, peak_kind)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (uniform random records, device RNG)",
                "config": config(n, world, prec_name), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks, "impl": "b200", "scatter_back": scatter}
        line.update(extras)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


FP32_LANES_PER_SM = 128  # FFMA lanes per SM (B200): FP32 peak = SMs x 128 x 2 flop x clock


def fp32_peak_tflops(clock_mhz=None):
    import torch
    props = torch.cuda.get_device_properties(0)
    mhz = clock_mhz or 1965.0
    return props.multi_processor_count * FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12


def ncu_metrics(name):
    """Per-kernel ncu metrics committed under profiles/ (issue activity, SIMD
    efficiency, L2 hit rate, occupancy); None when not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "kernel_metrics.json")) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def compute_roofline(kernel, pairs, flops_per_pair, ms, metrics_key):
    """Useful-flop roofline of an issue-bound pair loop: in-support pairs x
    flops per pair / kernel time against the FP32 (non-tensor) peak."""
    ach = pairs * flops_per_pair / (ms * 1e-3) / 1e12
    peak = fp32_peak_tflops()
    rl = {"bound": "fp32 issue (FFMA + MUFU, no tensor-core contraction)", "achieved": ach, "peak": peak,
          "unit": "TFLOP/s", "frac": ach / peak, "kernel": kernel, "flops_per_pair": flops_per_pair,
          "pairs_per_s": pairs / (ms * 1e-3),
          "peak_kind": "148 SMs x 128 FFMA lanes x 2 flop x 1965 MHz (B200 max SM clock)", "traffic": None}
    m = ncu_metrics(metrics_key)
    if m:
        rl["ncu"] = m
    return rl


def run_extras(args, world, rank, peak, peak_kind):
    """The other BASELINE configs and the paper's measurements, as extra keys
    of the default line.  N=1: everything; N>1: the sharded C5 only (all
    ranks take part)."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "benchmarks"))
    import workloads as W
    ex = {}

    def guard(name, fn, into=ex):
        t0 = time.time()
        try:
            r = fn()
        except Exception as e:  # reported, never fatal
            r = {"unavailable": "%s: %s" % (type(e).__name__, str(e)[:300])}
        r["bench_seconds"] = round(time.time() - t0, 2)
        into[name] = r
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    threads = os.cpu_count() or 1
    sub = argparse.Namespace(**vars(args))
    sub.steps, sub.warmup = min(args.steps, 10), max(3, min(args.warmup, 3))
    if world == 1:
        configs = {}

        def c1():
            r = W.c1(sub, peak, peak_kind)
            if not args.no_cpu:
                rate, secs = cpu_c1_rate(1 << 20, threads)
                r["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                                     "sample": "the full C1 workload: the reference's kick then drift on 1M "
                                               "default-AoS particles, %.3f s" % secs}
            return r

        def c3():
            r = W.c3(sub, peak, peak_kind)
            k = r["kernels"]
            pairs = k["fp32"]["pairs_in_support"]
            r["roofline"] = compute_roofline("k_pairs_c (fp32, reach %d)" % args.refine, pairs, 24,
                                             k["fp32"]["density_ms"], "pairs_c3_fp32")
            r["roofline_force"] = compute_roofline("k_force_c (fp32)", pairs, 40, k["force_fp32"]["force_ms"],
                                                   "force_c3_fp32")
            if "step_fp32" in k:
                r["roofline_force_masked"] = compute_roofline(
                    "k_force_masked (fp32, after a density that marked the in-support pairs)", pairs, 40,
                    k["step_fp32"]["force_masked_ms"], "force_masked_c3_fp32")
            r["hbm_frac_fp32"] = k["fp32"]["hbm_GBps_algorithmic"] / peak
            if not args.no_cpu:
                rate, secs = cpu_reference_kernels_rate(1 << 20, ["density"], threads, T=32, layout="soa")
                r["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                                     "sample": "the reference's own density_kernel (64-particle buffers, "
                                               "binary64, 64 pairs per particle) on a 1M-particle T=32 SoA, "
                                               "%d threads, %.2f s" % (threads, secs)}
                prate, psecs = cpu_c3_port_rate(1 << 22)
                r["cpu_baseline"]["port_cell_linked"] = {
                    "value": prate, "cores": 1, "kind": "port",
                    "sample": "cell-linked density of the oracle's C restatement, 65536 particles at C3's "
                              "density and h, one core, %.2f s" % psecs}
            return r

        def c4():
            pk = W.pcie_peaks()
            r = W.c4(sub, peak, peak_kind)
            ach = r["roofline"]["achieved"]
            r["roofline"].update({"peak": pk["bidirectional_GBps"], "frac": ach / pk["bidirectional_GBps"],
                                  "peak_kind": "measured: " + pk["method"]})
            r["pcie"] = pk
            if not args.no_cpu:
                rate, secs = cpu_c1_rate(1 << 22, threads, kernels=("drift",))
                r["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                                     "sample": "extrapolated per particle: the reference's drift step on a "
                                               "4M-particle host AoS (no transfers), %.3f s" % secs}
            return r

        guard("c1", c1, configs)
        guard("c3", c3, configs)
        guard("c4", c4, configs)
        ex["configs"] = configs
        guard("soa_vs_aos", lambda: W.soa_vs_aos(sub))
        guard("transform", lambda: W.transform_placement(sub, ROOT))
        guard("timestep", lambda: W.timestep_pipeline(sub))
    guard("sharded_c5", lambda: sharded_c5(sub, world, rank, peak, peak_kind))
    return ex


def sharded_c5(args, world, rank, peak, peak_kind):
    """C5 (BASELINE configs[4]): the 128M-particle reference timestep
    (density, force, kick, drift, migrate) sharded by x-slabs of cells over
    the ranks; time = max over ranks, strong scaling."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "benchmarks"))
    import workloads as W
    res = W.c5(args, peak, peak_kind, world, rank)
    keys = sorted(k for k, v in res["phases_ms"].items() if isinstance(v, float))
    t = torch.tensor([res["ms_per_step"]] + [res["phases_ms"][k] for k in keys], device="cuda",
                     dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    phases = {k: float(v) for k, v in zip(keys, t[1:].tolist())}
    n = args.c5_n
    out = {"value": n / (ms * 1e-3), "unit": "particle updates/s (full timesteps)", "ms_per_step": ms,
           "n_gpus": world, "scaling": "strong", "particles_total": n, "particles_rank0": res["particles_local"],
           "phases_ms_max_over_ranks": phases, "config": res["config"],
           "halo": "peer: each rank reads its +-1 neighbours' packed cell blocks in place through CUDA IPC "
                   "peer pointers (NVLink); no ghost copy, no NCCL on the data path" if world > 1 else
                   "none (one slab)", "migrated_per_step": res.get("sent_per_step")}
    # compute rooflines of the two pair kernels (uniform particles: 64 in-support neighbours by construction)
    pairs = 64.0 * n / world
    if phases.get("force"):
        out["roofline"] = compute_roofline("pack + k_force_masked (fp32, per rank: the in-support pairs the density marked)", pairs, 40, phases["force"], "force_c5")
    if phases.get("density"):
        out["roofline_density"] = compute_roofline("bin + pack + k_pairs_c with window masks (fp32, per rank)", pairs, 24,
                                                   phases["density"], "pairs_c5")
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rate, secs = cpu_reference_kernels_rate(1 << 18, ["density", "force", "kick", "drift"], threads, T=32,
                                                layout="soa")
        out["cpu_baseline"] = {"value": rate, "unit": "particle updates/s (full timesteps)", "cores": threads,
                               "kind": "reference",
                               "sample": "the reference's own timestep (density, force, kick, drift; 64-particle "
                                         "buffers, binary64) on a 256K-particle T=32 SoA, %d threads, %.2f s"
                                         % (threads, secs)}
    return out


def other_arm(args):
    """--workload c1 | c3 | c4 | c5 (benchmarks/workloads.py)."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "benchmarks"))
    import workloads as W
    from paper_2512_05516_b200 import api

    world, rank, local = dist_init()
    peak, kind = peaks()
    sampler = ClockSampler(local)
    sampler.start()
    l0 = api.launch_count()
    if args.workload == "c5":
        res = W.c5(args, peak, kind, world, rank)
        ms = torch.tensor([res["ms_per_step"]], device="cuda", dtype=torch.float64)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        res["ms_per_step"] = float(ms.item())
        res["value"] = args.c5_n / (res["ms_per_step"] * 1e-3)
    else:
        res = getattr(W, args.workload)(args, peak, kind)
    launches = api.launch_count() - l0
    clocks = sampler.stop()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.workload in ("c1", "c3", "c4", "c5"):
        try:
            if args.workload == "c4":  # extrapolated per particle from a <= 16M sample
                threads = os.cpu_count() or 1
                rate, secs = cpu_c1_rate(1 << 22, threads, kernels=("drift",))
                cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": "extrapolated per particle: the reference's drift step on a 4M-particle host AoS "
                                 "(no transfers: the data is already where the CPU computes), %.3f s" % secs}
            elif args.workload == "c5":
                rate, secs = cpu_c3_port_rate(args.c5_n)
                cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
                       "sample": "extrapolated per particle: cell-linked density of the oracle's C restatement on "
                                 "65536 particles at C5's density and h (one core), %.2f s" % secs}
            elif args.workload == "c1":
                threads = os.cpu_count() or 1
                rate, secs = cpu_c1_rate(1 << 20, threads)
                cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": "the full C1 workload: kick then drift on 1M default-AoS particles, %.3f s" % secs}
            else:
                rate, secs = cpu_c3_port_rate(1 << 22)
                cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
                       "sample": "65536 particles at C3's density and h in a sub-box (fewer neighbours at its "
                                 "faces), cell-linked density of the oracle's C restatement, %.2f s" % secs}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "unavailable: %s" % ex}
    if rank == 0:
        line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
                "scaling": "strong" if args.workload == "c5" else "weak", "vs_baseline": None, "dtype": "f64" if
                args.workload in ("c1", "c4") else "f32", "data": "synthetic (uniform random, device RNG)",
                "config": res["config"], "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res.get("e2e"),
                "gpu_launches": launches, "clocks": clocks, "impl": "b200", "workload": args.workload}
        for k in ("kernels", "phases_ms", "particles_local"):
            if k in res:
                line[k] = res[k]
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def torchrun_argv(argv, n, port):
    """The command that re-runs this bench under torch.distributed.run with
    n ranks on this node (the driver's own launch form)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % n,
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def maybe_reexec(args, argv):
    """--gpus N > 1 outside torchrun: one rank per GPU via torch.distributed.run."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = torchrun_argv(argv, args.gpus, port)
        env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
                   NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
        return subprocess.call(cmd, env=env)
    return None


def build_parser():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--prec", choices=["fp16", "bf16"], default="fp16")
    ap.add_argument("--chunk", type=int, default=1 << 21)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-sample", type=int, default=1 << 21)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="C2 only: skip configs c1/c3/c4, sharded_c5, soa_vs_aos, transform, timestep")
    ap.add_argument("--table-particles", type=int, default=1 << 16)
    ap.add_argument("--workload", choices=["c1", "c2", "c3", "c4", "c5"], default="c2",
                    help="BASELINE.json config (default c2 = configs[1], the headline)")
    ap.add_argument("--c4-n", type=int, default=1 << 26)
    ap.add_argument("--c5-n", type=int, default=1 << 27)
    ap.add_argument("--refine", type=int, default=2,
                    help="C3/C5 binning cells per density cell side (searched with reach = refine)")
    return ap


def main():
    argv = sys.argv[1:]
    args = build_parser().parse_args(argv)
    rc = maybe_reexec(args, argv)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return reference_arm(args)
    if args.workload != "c2":
        return other_arm(args)
    return b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
