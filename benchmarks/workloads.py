"""The non-default BASELINE.json configs as bench.py workloads (`--workload`).

  c1  kick / drift on 1M particles, AoS full-precision storage, in place
      (92 MB < L2: L2 flushed between timed launches, each launch timed alone)
  c3  SPH density, cell-linked, 4M uniform particles, SoA fp32 vs fp16 vs bf16
  c4  64M host-resident particles: streamed (narrowed 2-D DMA) vs managed vs
      in-place (whole records), one drift and one kick+drift step each
  c5  128M particles, density + kick/drift sharded by cell (NCCL halo)

Each returns the same JSON-line dict as the default C2 workload.
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
    kern = {"kick": "k_update_rec_multi (in-place kick, AoS f32 lanes)",
            "drift": "k_update_rec (in-place drift, AoS f64 x / f32 v)",
            "kick,drift": "k_update_rec_seq (kick then drift in one pass over the records)"}
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
    return {"value": n / (ms * 1e-3), "ms_per_step": ms, "roofline": out["kick,drift"]["roofline"],
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
        rl["note"] = ("issue-bound: ncu smsp__issue_active ~82% with ~56% SIMD efficiency and ~2.75 evaluated "
                      "candidates per in-support pair (profiles/r01_pairs_ncu_summary.txt); frac is on HBM bytes, "
                      "which are not the limiter")
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
            out["%s:%s" % (kernels, name)] = {"ms": s * 1e3, "value": n / s, "h2d_bytes": m["h2d_bytes"],
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
    from paper_2512_05516_b200.sharded import ShardedState, Slab, grid_for
    n = args.c5_n
    h, nc, cell = grid_for(n)
    slab = Slab(nc, cell, rank, world)
    st = ShardedState(n, slab, prec=32, h=h, reorder_every=args.c5_reorder)
    st.sort_by_cell()  # particles start in cell order; --c5-reorder k keeps them there every k-th step
    for _ in range(max(1, min(args.warmup, 2))):
        st.full_step(group=group) if args.c5_full else st.step(group=group)
    torch.cuda.synchronize()
    phases = {"kick_drift": [], "migrate": [], "density": [], "reorder": []}
    if args.c5_full:
        phases["force"] = []
    times = []
    for _ in range(max(2, min(args.steps, 5))):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        if args.c5_full:  # the reference's timestep order: density, force, kick+drift, migrate
            st.density(group)
            ev[1].record()
            st.force(group)
            ev[2].record()
            st.maybe_reorder()
            ev[3].record()
            st.kick_drift()
            ev[4].record()
            st.migrate(group)
            ev[5].record()
            ev[5].synchronize()
            phases["density"].append(ev[0].elapsed_time(ev[1]))
            phases["force"].append(ev[1].elapsed_time(ev[2]))
            phases["reorder"].append(ev[2].elapsed_time(ev[3]))
            phases["kick_drift"].append(ev[3].elapsed_time(ev[4]))
            phases["migrate"].append(ev[4].elapsed_time(ev[5]))
            times.append(ev[0].elapsed_time(ev[5]))
            continue
        st.kick_drift()
        ev[1].record()
        st.migrate(group)
        ev[2].record()
        st.density(group)
        ev[3].record()
        st.maybe_reorder()
        ev[4].record()
        ev[4].synchronize()
        phases["kick_drift"].append(ev[0].elapsed_time(ev[1]))
        phases["migrate"].append(ev[1].elapsed_time(ev[2]))
        phases["density"].append(ev[2].elapsed_time(ev[3]))
        phases["reorder"].append(ev[3].elapsed_time(ev[4]))
        times.append(ev[0].elapsed_time(ev[4]))
    ms = sum(times) / len(times)
    # one more step with sub-phase events (not part of the timed mean)
    import paper_2512_05516_b200.sharded as SH
    SH.PHASES.clear()
    SH.PHASES["_on"] = True
    st.step(group=group)
    torch.cuda.synchronize()
    ev = SH.PHASES.pop("_events", [])
    SH.PHASES.clear()
    sub = {}
    for (a, ea), (_, eb) in zip(ev, ev[1:]):
        sub[a] = sub.get(a, 0.0) + ea.elapsed_time(eb)
    phases["density_sub"] = [sub]
    return {"value": n / (ms * 1e-3), "ms_per_step": ms, "local_ms": ms,
            "roofline": {"bound": "compute (density)", "achieved": None, "peak": peak, "unit": "GB/s",
                         "frac": None, "kernel": "k_pairs_c + k_update_soa (kick/drift)"},
            "config": {"workload": "C5 (BASELINE configs[4]): %dM-particle density + %skick/drift sharded by cell "
                                   "with NCCL halo exchange" % (n >> 20, "force + " if args.c5_full else ""),
                       "particles_total": n, "step": "full (density, force, kick, drift, migrate)" if args.c5_full
                       else "kick, drift, migrate, density",
                       "cells_per_side": nc, "h": h, "storage": "SoA binary32 (default schema, T=32)"},
            "phases_ms": {k: (sum(v) / len(v) if k != "density_sub" else v[0]) for k, v in phases.items()},
            "particles_local": st.n}
