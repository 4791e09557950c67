"""C4 managed-memory orchestration variants (64M default-schema records,
drift step: gather + drift + scatter-back on every record), timed with CUDA
events.  Each variant moves the same bytes; only the migration policy
differs:

  prefetch_chunk     per chunk: prefetch to GPU, kernels, prefetch back
                     (sf_b200_run_host mode 1), on 3 rotating streams
  prefetch_chunk_na  the same without cudaMemAdvise
  prefetch_bulk      one prefetch of the whole range to the GPU, kernels per
                     chunk, one prefetch back
  prefetch_split     H2D prefetches on one stream, kernels on a second,
                     D2H prefetches on a third (event-chained per chunk)
  pinned_inplace     the pinned whole-record DMA reference (mode 2)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "benchmarks"))

import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import workloads as W  # noqa: E402
from paper_2512_05516_b200 import api  # noqa: E402

N = int(os.environ.get("N", str(1 << 26)))
CHUNK = int(os.environ.get("CHUNK", str(1 << 21)))


def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(str(r))
    return r


def loc(dev):
    try:
        l = rt.cudaMemLocation()
        l.type = rt.cudaMemLocationType.cudaMemLocationTypeDevice if dev >= 0 else \
            rt.cudaMemLocationType.cudaMemLocationTypeHost
        l.id = max(dev, 0)
        return l
    except Exception:
        return None


def prefetch(ptr, nbytes, dev, stream):
    # CUDA 12.x: cudaMemPrefetchAsync(ptr, count, dstDevice, stream); cudaCpuDeviceId = -1
    chk(rt.cudaMemPrefetchAsync(ptr, nbytes, dev, stream))


def main():
    P, v, src = W.random_default_aos(N)
    dst = api.View(P, CHUNK, "soa", "drift", 16)
    out = api.PackedBuffer.empty(dst)
    managed = api.HostBuffer(v.nbytes, 1)
    pinned = api.HostBuffer(v.nbytes, 0)
    for hb in (managed, pinned):
        t = torch.from_numpy(hb.numpy())
        for b in range(0, v.nbytes, 1 << 30):
            t[b:b + (1 << 30)].copy_(src.data[b:min(v.nbytes, b + (1 << 30))])
    torch.cuda.synchronize()
    del src
    torch.cuda.empty_cache()
    base = managed.ptr.value
    rb = 88
    chunks = [(r0, min(CHUNK, N - r0)) for r0 in range(0, N, CHUNK)]
    streams = [torch.cuda.Stream() for _ in range(3)]
    cv = api.View(P, CHUNK, "aos")
    res = {}

    def chunk_tensor(r0, cnt):
        class _I:
            __cuda_array_interface__ = {"shape": (cnt * rb,), "typestr": "|u1", "data": (base + r0 * rb, False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(_I(), device="cuda")

    def kernels(r0, cnt):
        view = cv if cnt == CHUNK else api.View(P, cnt, "aos")
        dv = dst if cnt == CHUNK else api.View(P, cnt, "soa", "drift", 16)
        buf = api.PackedBuffer(view, chunk_tensor(r0, cnt))
        o = out if cnt == CHUNK else api.PackedBuffer.empty(dv)
        api.gather_kernel(buf, dv, "drift", 1e-3, out=o)
        api.widen_merge(o, buf, "drift")

    def run(name, body, reps=3):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            body()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        s = min(ts)
        res[name] = {"ms": s * 1e3, "GBps_both_ways": 2 * v.nbytes / s / 1e9, "GBps_one_way": v.nbytes / s / 1e9,
                     "all_ms": [t * 1e3 for t in ts]}
        print(name, json.dumps(res[name]), flush=True)

    def prefetch_chunk(advise):
        def body():
            if advise:
                chk(rt.cudaMemAdvise(base, v.nbytes, rt.cudaMemoryAdvise.cudaMemAdviseSetPreferredLocation, -1))
                chk(rt.cudaMemAdvise(base, v.nbytes, rt.cudaMemoryAdvise.cudaMemAdviseSetAccessedBy, 0))
            for k, (r0, cnt) in enumerate(chunks):
                s = streams[k % 3]
                with torch.cuda.stream(s):
                    prefetch(base + r0 * rb, cnt * rb, 0, s.cuda_stream)
                    kernels(r0, cnt)
                    prefetch(base + r0 * rb, cnt * rb, -1, s.cuda_stream)
        return body

    def prefetch_bulk():
        s = torch.cuda.current_stream()
        prefetch(base, v.nbytes, 0, s.cuda_stream)
        for r0, cnt in chunks:
            kernels(r0, cnt)
        prefetch(base, v.nbytes, -1, s.cuda_stream)

    def prefetch_split():
        h2d, comp, d2h = streams
        for r0, cnt in chunks:
            e1, e2 = torch.cuda.Event(), torch.cuda.Event()
            prefetch(base + r0 * rb, cnt * rb, 0, h2d.cuda_stream)
            e1.record(h2d)
            comp.wait_event(e1)
            with torch.cuda.stream(comp):
                kernels(r0, cnt)
            e2.record(comp)
            d2h.wait_event(e2)
            prefetch(base + r0 * rb, cnt * rb, -1, d2h.cuda_stream)

    def migrate_only(dev):
        def body():
            s = torch.cuda.current_stream()
            prefetch(base, v.nbytes, dev, s.cuda_stream)
        return body

    def migrate_chunks(dev):
        def body():
            for k, (r0, cnt) in enumerate(chunks):
                prefetch(base + r0 * rb, cnt * rb, dev, streams[k % 3].cuda_stream)
        return body

    def pinned_inplace():
        api.run_host(v, pinned, api.View(P, N, "soa", "drift", 16), "drift", 1e-3, chunk=CHUNK, mode=2)

    def managed_mode1():
        api.run_host(v, managed, api.View(P, N, "soa", "drift", 16), "drift", 1e-3, chunk=CHUNK, mode=1)

    run("pinned_inplace", pinned_inplace)
    # pure page migration, no kernels: the limiter of every managed variant
    for rep in range(2):
        run("migrate_whole_to_gpu_%d" % rep, migrate_only(0), reps=1)
        run("migrate_whole_to_host_%d" % rep, migrate_only(-1), reps=1)
    for rep in range(2):
        run("migrate_chunks_to_gpu_%d" % rep, migrate_chunks(0), reps=1)
        run("migrate_chunks_to_host_%d" % rep, migrate_chunks(-1), reps=1)
    run("run_host_mode1", managed_mode1)
    run("prefetch_chunk", prefetch_chunk(True))
    run("prefetch_chunk_na", prefetch_chunk(False))
    run("prefetch_split", prefetch_split)
    run("prefetch_bulk", prefetch_bulk)
    print(json.dumps({"N": N, "chunk": CHUNK, "bytes_each_way": v.nbytes, "results": res}))


if __name__ == "__main__":
    main()
