"""The non-default BASELINE.json configs as bench.py workloads (`--workload`).

  c1  kick / drift on 1M particles, AoS full-precision storage, in place
      (92 MB < L2: L2 flushed between timed launches, each launch timed alone)
  c3  SPH density, cell-linked, 4M uniform particles, SoA fp32 vs fp16 vs bf16
  c4  64M host-resident particles: streamed (zero copy, narrowed lanes) vs managed vs
      in-place (whole records), one drift and one kick+drift step each
  c5  128M particles, density + kick/drift sharded by cell (peer-block halo)

plus the paper's three measurements on the B200 (bench.py puts them in the
default line): soa_vs_aos (kernel speedups), transform
(conversion placement host vs device) and timestep
(in-place vs streaming whole timestep over real PCIe).
"""
from __future__ import annotations

import math
import os
import time

import torch

from paper_2512_05516_b200 import api

UNIT = "particle updates/s"
L2_FLUSH_BYTES = 512 << 20


class L2Flush:
    """Write a buffer larger than L2, then read a second one: the write evicts
    the workload's lines, the read evicts the flush's own dirty lines, so the
    timed kernel starts with a cold L2 and does not pay the flush's
    write-back."""

    def __init__(self):
        self.buf = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
        self.rd = torch.ones(L2_FLUSH_BYTES // 8, dtype=torch.int64, device="cuda")

    def __call__(self):
        self.buf.fill_(1)
        self.rd.max()


def timed_each(fn, steps, flush=None, stream=None):
    """Per-launch CUDA-event times (ms), L2 flushed before each launch.  All
    launches are queued before the single synchronize, so host-side launch
    work overlaps the previous flush instead of landing inside a timed gap."""
    stream = stream or torch.cuda.current_stream()
    evs = []
    for _ in range(steps):
        if flush:
            flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def random_default_aos(n, seed=1234):
    P = api.Schema.default()
    v = api.View(P, n, "aos")
    src = api.PackedBuffer.empty(v)
    rec = src.data[: v.nbytes].view(n, 88)
    g = torch.Generator(device="cuda").manual_seed(seed)
    step = 1 << 22
    for b in range(0, n, step):
        e = min(n, b + step)
        m = e - b
        f = torch.rand(m, 17, device="cuda", generator=g)
        rec[b:e, 0:24] = f[:, 0:3].double().contiguous().view(torch.uint8).view(m, 24)
        rec[b:e, 24:32] = torch.arange(b, e, device="cuda", dtype=torch.int64).view(torch.uint8).view(m, 8)
        f[:, 3:6] = f[:, 3:6] * 2 - 1
        f[:, 13:17] = f[:, 13:17] * 2 - 1   # a, du ~ U(-1, 1): kick is not a no-op
        rec[b:e, 32:88] = f[:, 3:17].contiguous().view(torch.uint8).view(m, 56)
    return P, v, src


def roofline(bytes_per_unit, units, ms, peak, kind, kernel, traffic=None):
    ach = bytes_per_unit * units / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "peak_kind": kind, "kernel": kernel, "algorithmic_bytes_per_particle": bytes_per_unit,
            "traffic": traffic}


# ----------------------------------------------------------------------- C1
def c1(args, peak, peak_kind):
    n = 1 << 20
    P, v, src = random_default_aos(n)
    nat = api.convert(src, api.View(P, n, "aos", None, api.SF_PREC_NATIVE))
    # rotation set: 6 copies (554 MB > 126 MB L2), so every launch finds its buffer cold
    rot = [api.convert(src, api.View(P, n, "aos", None, api.SF_PREC_NATIVE)) for _ in range(6)]
    flush = L2Flush()
    kern = {"kick": "k_update_rec_tile<128> (in-place kick on the AoS records, TMA-staged)",
            "drift": "k_update_rec_tile<128> (in-place drift on the AoS records, TMA-staged)",
            "kick,drift": "k_update_rec_tile<128> (kick then drift in one pass over the records)"}
    out = {}
    # algorithmic bytes: kick reads v,a,u,du (32 B) writes v,u (16 B); drift reads x,v (36 B) writes x (24 B);
    # the one-pass sequence reads x,v,a,u,du (56 B) and writes x,v,u (40 B)
    for k, bpp in (("kick", 48), ("drift", 60), ("kick,drift", 96)):
        fn = lambda: api.run_kernel(nat, k, 1e-3, buffer_size=64)  # noqa: E731
        for _ in range(args.warmup):
            fn()
        t = timed_each(fn, args.steps, flush)
        ms_f = sum(t) / len(t)
        # back-to-back launches over the rotation set, one event pair
        reps = max(args.steps, 12)
        for b in rot:
            api.run_kernel(b, k, 1e-3, buffer_size=64)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for r in range(reps):
            api.run_kernel(rot[r % len(rot)], k, 1e-3, buffer_size=64)
        e.record()
        e.synchronize()
        ms_r = a.elapsed_time(e) / reps
        ms = min(ms_f, ms_r)
        out[k] = {"ms": ms, "ms_flushed_each": ms_f, "ms_rotating_cold": ms_r, "value": n / (ms * 1e-3),
                  "roofline": roofline(bpp, n, ms, peak, peak_kind, kern[k])}
    ms = out["kick,drift"]["ms"]
    # end to end: the 1M records in pinned host memory, whole records H2D, gather to the full-precision SoA +
    # kick + drift + scatter-back, whole records D2H (sf_b200_run_host in place, 3-stream chunk ring)
    hb = api.HostBuffer(v.nbytes, 0)
    torch.from_numpy(hb.numpy()).copy_(src.data[: v.nbytes])
    torch.cuda.synchronize()
    dst = api.View(P, n, "soa", None, api.SF_PREC_NATIVE)
    api.run_host(v, hb, dst, "kick,drift", 1e-3, chunk=1 << 18, mode=2)
    secs = []
    for _ in range(max(3, min(args.steps, 10))):
        m = api.run_host(v, hb, dst, "kick,drift", 1e-3, chunk=1 << 18, mode=2)
        secs.append(m["seconds"])
    hb.free()
    e2e_s = sum(secs) / len(secs)
    e2e = {"value": n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": m["h2d_bytes"], "d2h_bytes_per_step": m["d2h_bytes"],
           "ms": e2e_s * 1e3, "path": "sf_b200_run_host(mode 2): pinned host AoS, whole records H2D || gather to the "
                                      "full-precision SoA + kick + drift + scatter-back || whole records D2H"}
    return {"value": n / (ms * 1e-3), "ms_per_step": ms, "roofline": out["kick,drift"]["roofline"], "e2e": e2e,
            "config": {"workload": "C1 (BASELINE configs[0]): kick then drift in place on 1M particles, AoS "
                                   "full-precision storage (default 88-B schema), one pass over the records "
                                   "(run_kernel('kick,drift'); the per-kernel launches are under 'kernels')", "particles": n,
                       "l2": "92 MB < 126 MB L2.  Two timings, the faster reported: (a) L2 flushed before every "
                             "timed launch (512 MB write, then a 512 MB read so the flush's dirty lines are written "
                             "back before the timed region), (b) back-to-back launches rotating over 6 copies "
                             "(554 MB > L2, each launch's buffer cold in L2)",
                       "arith": "binary64, bit-exact vs reference"},
            "kernels": out}


# ----------------------------------------------------------------------- C3
def c3(args, peak, peak_kind):
    from paper_2512_05516_b200.sharded import grid_for
    n = 1 << 22
    h, nc, cell = grid_for(n)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float32)
    m = torch.full((n,), 1.0 / n, device="cuda")
    hh = torch.full((n,), h, device="cuda")
    refine = args.refine            # binning cells of side 1/(refine nc) >= 2h/refine, searched with reach = refine
    fine = cell / refine
    dims = (nc * refine,) * 3
    out = {}
    for name, prec, dt in (("fp32", api.SF_PREC_NATIVE, torch.float32), ("fp16", 16, torch.float16),
                           ("bf16", api.SF_PREC_BF16, torch.bfloat16)):
        xs, ms_, hs = x.to(dt), m.to(dt), hh.to(dt)
        xf = xs.float().contiguous()
        cs, perm = api.bin_particles(xf, (0, 0, 0), fine, dims)
        rho = torch.empty(n, device="cuda")
        fn = lambda: api.density_cells(xs, ms_, hs, cs, perm, (0, 0, 0), fine, dims, reach=refine,  # noqa: E731
                                       prec=prec, rho=rho)
        for _ in range(args.warmup):
            fn()
        t = timed_each(fn, max(3, args.steps // 5))
        fb = lambda: api.bin_particles(xf, (0, 0, 0), fine, dims, cell_start=cs, perm=perm)  # noqa: E731
        fb()  # scratch allocation outside the timed launches
        tb = timed_each(fb, max(3, args.steps // 5))
        msd, msb = sum(t) / len(t), sum(tb) / len(tb)
        # pairs inside the support, for pairs/s
        pairs = None
        if name == "fp32":  # neighbours inside 2h, sampled (256 particles x all, in chunks)
            cnt = 0
            for b in range(0, n, 1 << 20):
                cnt += int((torch.cdist(x[:256], x[b:b + (1 << 20)]) < 2 * h).sum().item())
            pairs = cnt / 256 * n
        bytes_pp = {"fp32": 24, "fp16": 12, "bf16": 12}[name]
        out[name] = {"density_ms": msd, "bin_ms": msb, "value": n / (msd * 1e-3),
                     "hbm_GBps_algorithmic": bytes_pp * n / (msd * 1e-3) / 1e9,
                     "pairs_in_support": pairs}
        if name == "fp32":
            # cell-linked force on the same particles: rho from the density
            # just computed, P from the EOS at u = 1 (P = (gamma - 1) rho u), random velocities
            vel = torch.rand(n, 3, generator=g, device="cuda") * 2 - 1
            pres = rho * (2.0 / 3.0)
            acc, dudt = torch.empty(n, 3, device="cuda"), torch.empty(n, device="cuda")
            ff = lambda: api.force_cells(xs, vel, ms_, hs, rho, pres, cs, perm, (0, 0, 0), fine, dims,  # noqa: E731
                                         reach=refine, prec=prec, a=acc, du=dudt)
            for _ in range(args.warmup):
                ff()
            tf = timed_each(ff, max(3, args.steps // 5))
            msf = sum(tf) / len(tf)
            out["force_fp32"] = {"force_ms": msf, "value": n / (msf * 1e-3),
                                 "pairs_in_support_per_s": pairs / (msf * 1e-3),
                                 "note": "pack (x,h | v,m | P/rho^2) + k_force_c; includes the rho == 0 check "
                                         "(one stream sync)"}
            if refine <= 2:
                # one SPH step's density then force sharing the pair search (block API, window masks): the
                # density marks every home's in-support pairs, the force evaluates exactly those
                pos = torch.empty(n, 4, device="cuda")
                hsb = torch.empty(n, device="cuda")
                hmx = torch.zeros(4, dtype=torch.int32, device="cuda")
                api.cells_pack(xs, ms_, hs, perm, pos, hsb, hmx, prec=prec)
                blk = api.cell_block(pos, hsb, cs, hmx, 0, dims[0], 0.0)
                mk = api.window_masks(n, refine)
                geo = (n, perm, (0.0, 0.0), fine, dims[0], dims[1], dims[2])
                rho2 = torch.empty(n, device="cuda")
                fdm = lambda: api.density_cells_blocks([blk], *geo, reach=refine, rho=rho2, masks=mk)  # noqa: E731
                fdp = lambda: api.density_cells_blocks([blk], *geo, reach=refine, rho=rho2)  # noqa: E731
                for _ in range(args.warmup):
                    fdp()
                    fdm()
                tdp = timed_each(fdp, max(3, args.steps // 5))
                tdm = timed_each(fdm, max(3, args.steps // 5))
                velb = torch.empty(n, 4, device="cuda")
                api.force_pack(vel, rho2, rho2 * (2.0 / 3.0), perm, velb)
                fbk = api.force_block(pos, velb, hsb, cs, hmx, 0, dims[0], 0.0)
                a2, du2 = torch.empty(n, 3, device="cuda"), torch.empty(n, device="cuda")
                ffm = lambda: api.force_cells_blocks([fbk], *geo, reach=refine, a=a2, du=du2, masks=mk)  # noqa: E731
                for _ in range(args.warmup):
                    ffm()
                tfm = timed_each(ffm, max(3, args.steps // 5))
                mdp, mdm, mfm = (sum(t_) / len(t_) for t_ in (tdp, tdm, tfm))
                out["step_fp32"] = {
                    "density_pairs_ms": mdp, "density_pairs_masked_ms": mdm, "force_masked_ms": mfm,
                    "density_then_force_ms": mdm + mfm,
                    "pairs_in_support_per_s_force": pairs / (mfm * 1e-3),
                    "note": "pair kernels only (the block API: bin and pack done once outside): k_pairs_c, "
                            "k_pairs_c writing window masks, then k_force_masked over the marked pairs; "
                            "compare density_pairs_ms + the window-sweep force"}
    ms = out["fp32"]["density_ms"]
    rl = {"bound": "issue (FP32 + MUFU)", "achieved": out["fp32"]["hbm_GBps_algorithmic"], "peak": peak,
          "unit": "GB/s", "frac": out["fp32"]["hbm_GBps_algorithmic"] / peak, "peak_kind": peak_kind,
          "kernel": "k_pairs_c (fp32, reach %d)" % refine, "algorithmic_bytes_per_particle": 24, "traffic": None}
    if out["fp32"]["pairs_in_support"]:
        rl["pairs_per_s"] = out["fp32"]["pairs_in_support"] / (ms * 1e-3)
        # the limiter is instruction issue, not bytes: useful FP32 work against the FP32 (non-tensor) peak
        props = torch.cuda.get_device_properties(0)
        peak_tf = props.multi_processor_count * 128 * 2 * 1.965e9 / 1e12  # FMA lanes x 2 flop x max SM clock
        rl["useful_TFLOPs"] = rl["pairs_per_s"] * 24 / 1e12  # ~24 flops per in-support pair
        rl["fp32_peak_TFLOPs"] = peak_tf
        rl["useful_flop_frac"] = rl["useful_TFLOPs"] / peak_tf
        rl["note"] = ("FP32-issue-bound pair loop: see the ncu issue activity, SIMD efficiency and FMA-pipe use "
                      "under roofline.ncu (profiles/kernel_metrics.json)")
    return {"value": n / (ms * 1e-3), "ms_per_step": ms, "roofline": rl,
            "config": {"workload": "C3 (BASELINE configs[2]): SPH density, cell-linked, 4M uniform particles, "
                                   "SoA fp32 vs fp16 vs bf16", "particles": n, "h": h, "cells_per_side": nc,
                       "binning_cells_per_side": nc * refine, "reach": refine,
                       "value_is": "fp32 density (pack + pair kernels); binning reported separately"},
            "kernels": out}


# ----------------------------------------------------------------------- C4
def c4(args, peak, peak_kind):
    n = args.c4_n
    P, v, src = random_default_aos(n)
    pinned = api.HostBuffer(v.nbytes, 0)
    managed = api.HostBuffer(v.nbytes, 1)
    hp, hm = pinned.numpy(), managed.numpy()
    step = 1 << 22
    for b in range(0, v.nbytes, step * 88):
        e = min(v.nbytes, b + step * 88)
        blk = src.data[b:e].cpu().numpy()
        hp[b:e] = blk
        hm[b:e] = blk
    del src
    torch.cuda.empty_cache()
    out = {}
    for kernels, dst_set in (("drift", "drift"), ("kick,drift", None)):
        dst = api.View(P, n, "soa", dst_set, 16)
        for mode, name, hb in ((0, "streamed", pinned), (1, "managed", managed), (3, "managed_mapped", managed),
                               (2, "inplace", pinned)):
            api.run_host(v, hb, dst, kernels, 1e-3, chunk=args.chunk, mode=mode)
            secs = []
            for _ in range(max(2, min(args.steps, 5))):
                m = api.run_host(v, hb, dst, kernels, 1e-3, chunk=args.chunk, mode=mode)
                secs.append(m["seconds"])
            s = sum(secs) / len(secs)
            out["%s:%s" % (kernels, name)] = {"ms": s * 1e3, "ms_min": min(secs) * 1e3, "ms_max": max(secs) * 1e3,
                                              "value": n / s, "h2d_bytes": m["h2d_bytes"],
                                              "d2h_bytes": m["d2h_bytes"],
                                              "pcie_GBps": (m["h2d_bytes"] + m["d2h_bytes"]) / s / 1e9}
    pinned.free()
    managed.free()
    best_mode = max(("streamed", "managed", "managed_mapped", "inplace"), key=lambda m: out["drift:" + m]["value"])
    best = out["drift:" + best_mode]
    return {"value": best["value"], "ms_per_step": best["ms"],
            "roofline": {"bound": "pcie", "achieved": best["pcie_GBps"], "peak": None, "unit": "GB/s",
                         "frac": None, "kernel": "run_host %s (k_gather_multi + scatter-merge, 3-stream chunk ring)" % best_mode},
            "config": {"workload": "C4 (BASELINE configs[3]): 64M host-resident particles, streamed vs managed "
                                   "vs in-place, one drift and one kick+drift step (gather, compute, scatter-back)",
                       "particles": n, "chunk": args.chunk, "soa_precision": "binary16",
                       "value_is": "drift step, best mode (%s)" % best_mode},
            "kernels": out}


# ----------------------------------------------------------------------- C5
def c5(args, peak, peak_kind, world, rank, group=None):
    """One rank of the C5 timestep through the C++ shard (sf_b200_shard_step):
    density, force, kick, drift, then migration, one library call per step;
    phase times from the library's own CUDA events (waits on the neighbours
    included)."""
    from paper_2512_05516_b200.sharded import ShardedState, Slab, grid_for
    n = args.c5_n
    h, nc, cell = grid_for(n)
    slab = Slab(nc, cell, rank, world)
    st = ShardedState(n, slab, prec=32, h=h, group=group, refine=args.refine)
    st.sort_by_cell()  # particles start in cell order; the shard's migration keeps the stayers in it
    st.stream("P").copy_(st.stream("rho") * (2.0 / 3.0) * st.stream("u"))  # EOS pressure, P = (gamma-1) rho u
    kernels = "density,force,kick,drift"
    for _ in range(max(1, min(args.warmup, 2))):
        st.full_step(1e-3, timed=True)
    torch.cuda.synchronize()
    runs = []
    for _ in range(max(2, min(args.steps, 5))):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        runs.append(st.full_step(1e-3, timed=True))
    keys = ["step_ms"] + [k + "_ms" for k in kernels.split(",")] + ["migrate_ms"]
    avg = {k: sum(r[k] for r in runs) / len(runs) for k in keys}
    phases = {"density": avg["density_ms"], "force": avg["force_ms"],
              "kick_drift": avg["kick_ms"] + avg["drift_ms"], "migrate": avg["migrate_ms"]}
    ms = avg["step_ms"]
    out = {"value": n / (ms * 1e-3), "ms_per_step": ms, "local_ms": ms,
           "roofline": {"bound": "compute (density, force)", "achieved": None, "peak": peak, "unit": "GB/s",
                        "frac": None, "kernel": "k_pairs_c + k_force_c"},
           "config": {"workload": "C5 (BASELINE configs[4]): %dM-particle density + force + kick/drift sharded by "
                                  "cell over %d GPU(s), halo read in place from the neighbours' blocks" % (n >> 20, world),
                      "particles_total": n, "step": "full reference timestep (density, force, kick, drift) + migration, "
                                                    "one sf_b200_shard_step call",
                      "cells_per_side": nc, "h": h, "storage": "SoA binary32 (default schema, T=32)",
                      "halo": "peer blocks over CUDA IPC (NVLink), device-side epoch ordering" if world > 1 else
                              "none (one slab)"},
           "phases_ms": phases, "particles_local": st.n, "sent_per_step": runs[-1]["sent"]}
    st.close()
    return out


# ----------------------------------------------------------------- PCIe probe
def pcie_peaks(nbytes: int = 1 << 30, reps: int = 3) -> dict:
    """Pinned cudaMemcpyAsync H2D, D2H and both directions at once (two
    streams), GB/s: the roofline denominators of the host-resident C4 step."""
    hb = api.HostBuffer(nbytes, 0)
    hb2 = api.HostBuffer(nbytes, 0)
    h1, h2 = torch.from_numpy(hb.numpy()), torch.from_numpy(hb2.numpy())
    d1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            dt_ = time.perf_counter() - t0
            best = dt_ if best is None else min(best, dt_)
        return best

    h2d = nbytes / timed(lambda: d1.copy_(h1, non_blocking=True)) / 1e9
    d2h = nbytes / timed(lambda: h1.copy_(d1, non_blocking=True)) / 1e9

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    bidir = 2 * nbytes / timed(both) / 1e9
    del d1, d2
    hb.free()
    hb2.free()
    return {"h2d_GBps": h2d, "d2h_GBps": d2h, "bidirectional_GBps": bidir,
            "method": "pinned cudaMemcpyAsync of %d MiB, best of %d; bidirectional = H2D and D2H on two "
                      "streams at once" % (nbytes >> 20, reps)}


# ----------------------------------------------------------- SoA vs AoS (paper Fig. compute)
def soa_vs_aos(args, n: int = 1 << 24) -> dict:
    """Kernel time on the unpacked AoS vs the SoA streams (the paper's
    compute-only comparison), 16M particles on the B200:
    kick and drift in place (k_update_rec_tile on records vs k_update_soa on
    streams) and the reference-semantics density (64-particle buffers,
    binary64, k_density_buffer), at the default precision (f64 x, f32 rest)
    and at T=16 (x kept at f64, the reference bench's exclusion)."""
    P, v, src = random_default_aos(n, seed=77)
    out = {}
    for label, prec, excl in (("default", api.SF_PREC_NATIVE, ""), ("T16", 16, "x")):
        aos = api.convert(src, api.View(P, n, "aos", None, prec, excl))
        soa = api.convert(src, api.View(P, n, "soa", None, prec, excl))
        for k, reps in (("kick", 10), ("drift", 10), ("density", 3)):
            row = {}
            for layout, buf in (("aos", aos), ("soa", soa)):
                fn = lambda: api.run_kernel(buf, k, 1e-3, buffer_size=64)  # noqa: E731
                fn()
                t = timed_each(fn, reps)
                row[layout + "_ms"] = sum(t) / len(t)
            row["soa_speedup"] = row["aos_ms"] / row["soa_ms"]
            out["%s/%s" % (k, label)] = row
        del aos, soa
    return {"particles": n, "rows": out,
            "paper": "SoA vs AoS kernel speedup: kick/drift ~8x GH200, ~4x H100; density ~4x on Nvidia "
                     "(PAPER.md:533)",
            "note": "compute only, inputs resident in HBM (1.4 GB AoS > L2), no transfers; kick/drift are "
                    "HBM-bound on both layouts (the AoS pass reads whole records once with one TMA bulk copy "
                    "per CTA), density is FP64-bound"}


# ----------------------------------------------------------- transform placement (paper Fig. transform)
def _lib_csv(lib_path, cmd, ints, strings):
    import ctypes as C
    L = C.CDLL(lib_path)
    L.sf_config_create.argtypes = [C.POINTER(C.c_void_p)]
    L.sf_config_set_int.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
    L.sf_config_set_string.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
    getattr(L, cmd).argtypes = [C.c_void_p, C.POINTER(C.c_char_p)]
    L.sf_config_destroy.argtypes = [C.c_void_p]
    L.sf_last_error.restype = C.c_char_p
    cfg = C.c_void_p()
    L.sf_config_create(C.byref(cfg))
    for k, val in ints.items():
        L.sf_config_set_int(cfg, k.encode(), val)
    for k, val in strings.items():
        L.sf_config_set_string(cfg, k.encode(), val.encode())
    out = C.c_char_p()
    st = getattr(L, cmd)(cfg, C.byref(out))
    text = out.value.decode() if out.value else ""
    L.sf_config_destroy(cfg)
    if st != 0:
        raise RuntimeError(L.sf_last_error().decode())
    rows = [ln.split(",") for ln in text.splitlines() if ln and not ln.startswith("#")]
    return [dict(zip(rows[0], r)) for r in rows[1:]]


def transform_placement(args, root: str, n: int = 1 << 17) -> dict:
    """Where to run U.N.C (bench.cpp:214-267), measured:
    host placement = the unmodified reference's own CPU conversion
    (narrow_into + unpack_into + aos_to_soa_into, its `bench transform` host
    rows, single-threaded as in the reference) + a measured pinned H2D of the
    converted SoA bytes; device placement = a measured pinned H2D of the
    whole compressed AoS + the fused B200 gather.  ratio = host / device
    (the reference's definition with measured instead of modelled moves)."""
    import os
    ref_lib = os.path.join(root, "oracle", "_ref", "libsoaforge_ref.so")
    sets = ["full", "density", "force", "kick", "drift"]
    ref = _lib_csv(ref_lib, "sf_run_bench_transform", {"particles": n},
                   {"kernels": "density,force,kick,drift", "precision": "32,16"})
    host_conv = {(r["kernel"], int(r["precision"])): (float(r["convert_s"]), int(r["bytes_moved"]))
                 for r in ref if r["placement"] == "host"}
    schema = api.Schema.default()
    hb = api.HostBuffer(n * 200 + 4096, 0)
    hsrc = torch.from_numpy(hb.numpy())
    _, aos_v, src = random_default_aos(n, seed=5)

    def h2d_s(nbytes):
        d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        fn = lambda: d.copy_(hsrc[:nbytes], non_blocking=True)  # noqa: E731
        fn()
        t = timed_each(fn, 5)
        return min(t) * 1e-3

    rows = {}
    for T, prec in ((32, 32), (16, 16), ("bf16", api.SF_PREC_BF16)):
        # the reference's population at precision T: with_uniform_precision(S, T, {"x"}) stored compressed
        # (bench.cpp make_population); bf16 (no reference PrecisionSpec) gathers from the default AoS
        srcT = src if T == "bf16" else api.convert(src, api.View(schema, n, "aos", None, api.SF_PREC_PACKED + T, "x"))
        whole_s = h2d_s(srcT.view.nbytes)
        for name in sets:
            dv = api.View(schema, n, "soa", None if name == "full" else name, prec, "x")
            out = api.PackedBuffer.empty(dv)
            fn = lambda: api.gather(srcT, dv, out=out)  # noqa: E731
            fn()
            t = timed_each(fn, 10)
            dev_conv = min(t) * 1e-3
            row = {"device_convert_s": dev_conv, "device_move_s": whole_s, "device_bytes": srcT.view.nbytes,
                   "device_s": dev_conv + whole_s}
            if T != "bf16" and (name, T) in host_conv:
                hc, hbytes = host_conv[(name, T)]
                hm = h2d_s(hbytes)
                row.update({"host_convert_s": hc, "host_move_s": hm, "host_bytes": hbytes, "host_s": hc + hm,
                            "ratio": (hc + hm) / (dev_conv + whole_s)})
            rows["%s/%s" % (name, T)] = row
    hb.free()
    best16 = max(r["ratio"] for k, r in rows.items() if k.endswith("/16") and "ratio" in r)
    best32 = max(r["ratio"] for k, r in rows.items() if k.endswith("/32") and "ratio" in r)
    return {"particles": n, "rows": rows, "best_ratio_32": best32, "best_ratio_16": best16,
            "cpu_threads": 1,
            "paper": "GPU-side vs CPU-side transform: up to 35x (32-bit), 500x (16-bit) on GH200/MI300A "
                     "(PAPER.md:511)",
            "note": "x kept at f64 (bench.cpp's with_uniform_precision exclusion); host conversion = the "
                    "reference's own bench transform host rows (oracle/_ref, single-threaded like the "
                    "reference); moves measured over this box's PCIe"}


# ----------------------------------------------------------- whole timestep (paper Fig. pipeline)
def timestep_pipeline(args, n: int = 1 << 20) -> dict:
    """The paper's end-to-end question on a PCIe B200:
    one reference timestep (density, force, kick, drift; 64-particle buffers,
    binary64) on a host-resident AoS, through this library's
    sf_run_bench_pipeline with real transfers (pipelines.cpp:231-296
    semantics): dev-native = the AoS baseline (no transformation), dev-soa
    = the GPU-side AoS->SoA transformation; in-place = whole records once
    each way, streaming = each kernel's narrowed fields each way."""
    from paper_2512_05516_b200 import _lib
    cfg = {"kernels": "density,force,kick,drift", "variants": "dev-native,dev-soa", "modes": "inplace,streaming",
           "precision": "32,16"}
    # warm-up pass (module loading, pinned-allocation first touch): each row is one timed pass, as in the reference
    _lib_csv(_lib.LIB_PATH, "sf_run_bench_pipeline", {"particles": 1 << 14}, cfg)
    rows = _lib_csv(_lib.LIB_PATH, "sf_run_bench_pipeline", {"particles": n}, cfg)
    res = {}
    for r in rows:
        key = "%s/%s/%s" % (r["variant"], r["mode"], r["precision"])
        res[key] = {k: float(r[k]) for k in ("total_s", "convert_s", "move_s", "compute_s", "merge_s")}
        res[key].update({"bytes_to_device": int(r["bytes_to_device"]), "bytes_to_host": int(r["bytes_to_host"]),
                         "share_force": float(r["share_force"]), "share_density": float(r["share_density"])})
    speed = {}
    for mode in ("inplace", "streaming"):
        for prec in ("32", "16"):
            b = res.get("dev-native/%s/%s" % (mode, prec))
            t = res.get("dev-soa/%s/%s" % (mode, prec))
            if b and t:
                speed["%s/%s" % (mode, prec)] = b["total_s"] / t["total_s"]
    base = res.get("dev-native/inplace/32")
    if base:
        for mode in ("inplace", "streaming"):
            for prec in ("32", "16"):
                t = res.get("dev-soa/%s/%s" % (mode, prec))
                if t:
                    speed["%s/%s_vs_aos_inplace32" % (mode, prec)] = base["total_s"] / t["total_s"]
    return {"particles": n, "rows": res, "soa_speedup_vs_aos": speed,
            "paper": "In-place / Streaming vs AoS baseline: 2.6x / ~2x GH200, 1.9x / 1.4x H100 (PAPER.md:554)",
            "note": "moves are measured over PCIe: in place = pinned cudaMemcpy of the whole compressed records "
                    "each way; streaming = the conversion kernels read / store only the kernel's narrowed lanes "
                    "of the pinned host records in place (zero copy); phases run one after another as in the "
                    "reference's Run (not overlapped)"}
