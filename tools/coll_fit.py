"""Collective latency / bandwidth lines for the cost model's NCCL-vs-kernel
choice: every collective the executor emits, both implementations, a size
sweep, shards weighted by the bench's SM-cap ratios.  Run with torchrun (one
process per GPU):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/coll_fit.py --json out.json

Implementations (what Executor._use_p2p chooses between):
  all_gather      p2p = hap_p2p_all_gather_push   nccl = hap_all_gather_v (grouped send/recv)
  reduce_scatter  p2p = hap_p2p_reduce_scatter_direct   nccl = hap_reduce_scatter_v
  all_reduce      p2p = hap_p2p_all_reduce (two-shot)   nccl = hap_all_reduce
  all_to_all      p2p = hap_p2p_all_to_all (push)       nccl = hap_all_to_all_v
Each call is timed as 10 launches in one CUDA graph (no host launch cost),
max over ranks.  `x` = bytes of the full tensor (the cost model's
elements x bytes_per_element).  Kernel launches use the rank's SM cap, as the
executor does.  `python tools/coll_fit.py --fit a.json b.json ...` fits
cost_model.fit_linear per (world, op, impl) and writes
paper_2401_05965_b200/collectives_b200.json.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OPS = ("all_gather", "reduce_scatter", "all_reduce", "all_to_all")


def _register(L, ctx, t, world):
    import torch
    import torch.distributed as dist

    from paper_2401_05965_b200._lib import check, i64_array

    hb = ctypes.create_string_buffer(64)
    base, boff = ctypes.c_int64(), ctypes.c_int64()
    check(L.hap_p2p_buffer_handle(ctx, t.data_ptr(), hb, ctypes.byref(base), ctypes.byref(boff)))
    trip = [None] * world
    dist.all_gather_object(trip, (bytes(hb.raw), base.value, boff.value))
    ptrs = (ctypes.c_void_p * world)()
    check(L.hap_p2p_buffer_open(ctx, t.data_ptr(), b"".join(x[0] for x in trip), i64_array([x[1] for x in trip]),
                                i64_array([x[2] for x in trip]), ptrs))
    return torch.tensor([int(p or 0) for p in ptrs], dtype=torch.int64, device=t.device)


def bench(args):
    import torch
    import torch.distributed as dist

    from paper_2401_05965_b200 import workloads
    from paper_2401_05965_b200._lib import BF16, F32, check, i64_array, lib
    from paper_2401_05965_b200.executor import NcclGroup
    from paper_2401_05965_b200.sharding import offsets, round_shards

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    L = lib()
    group = NcclGroup.from_torch_distributed()
    caps = workloads.sm_caps(world)
    cap = caps[rank]
    ratios = [c / sum(caps) for c in caps]
    inner = 768
    stream = torch.cuda.Stream(dev)
    ctx = ctypes.c_void_p()
    check(L.hap_symm_create(ctypes.byref(ctx), 1 << 20, rank, world))
    h = ctypes.create_string_buffer(64)
    check(L.hap_symm_handle(ctx, h))
    handles = [None] * world
    dist.all_gather_object(handles, bytes(h.raw))
    check(L.hap_symm_open(ctx, b"".join(handles)))
    s = stream.cuda_stream
    results = []

    def timed(fn, name):
        for _ in range(3):
            check(fn(), name)
        torch.cuda.synchronize(dev)
        dist.barrier()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
            for _ in range(10):
                fn()
        torch.cuda.synchronize(dev)
        dist.barrier()
        with torch.cuda.stream(stream):
            graph.replay()
        torch.cuda.synchronize(dev)
        best = 1e30
        for _ in range(3):
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(args.reps):
                    graph.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            t = torch.tensor([e0.elapsed_time(e1) / (args.reps * 10)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            best = min(best, float(t.item()))
        del graph
        return best * 1e-3

    for rows in [int(v) for v in args.rows.split(",")]:
        sizes = round_shards(rows, ratios)
        offs = offsets(sizes)
        counts = [sz * inner for sz in sizes]
        devsz = torch.tensor([sizes, offs[:-1]], dtype=torch.int64, device=dev)
        carr = i64_array(counts)
        total_b16 = rows * inner * 2
        # ---- all-gather
        send = torch.randn(max(1, counts[rank]), device=dev).to(torch.bfloat16)
        out = torch.empty(rows * inner, device=dev, dtype=torch.bfloat16)
        outs = _register(L, ctx, out, world)
        impls = {
            "p2p": lambda: L.hap_p2p_all_gather_push(ctx, send.data_ptr(), outs.data_ptr(), BF16, 1, inner, rows,
                                                     devsz[0].data_ptr(), devsz[1].data_ptr(), rows * inner, cap, s),
            "nccl": lambda: L.hap_all_gather_v(group.comm, send.data_ptr(), out.data_ptr(), carr, BF16, 0, None, s),
        }
        for name, fn in impls.items():
            results.append({"op": "all_gather", "impl": name, "rows": rows, "bytes": total_b16,
                            "s": timed(fn, f"all_gather {name}")})
        # ---- reduce-scatter
        part = torch.randn(rows * inner, device=dev).to(torch.bfloat16)
        rs_out = torch.empty(max(1, counts[rank]), device=dev, dtype=torch.bfloat16)
        scratch = torch.empty(world * max(counts), device=dev, dtype=torch.bfloat16)
        parts = _register(L, ctx, part, world)
        impls = {
            "p2p": lambda: L.hap_p2p_reduce_scatter_direct(ctx, parts.data_ptr(), rs_out.data_ptr(), BF16, 1, inner,
                                                           rows, devsz[0].data_ptr(), devsz[1].data_ptr(),
                                                           counts[rank], cap, s),
            "nccl": lambda: L.hap_reduce_scatter_v(group.comm, part.data_ptr(), rs_out.data_ptr(), carr, BF16,
                                                   scratch.data_ptr(), s),
        }
        for name, fn in impls.items():
            results.append({"op": "reduce_scatter", "impl": name, "rows": rows, "bytes": total_b16,
                            "s": timed(fn, f"reduce_scatter {name}")})
        # ---- all-reduce (fp32, in place: the gradient buckets)
        n = rows * inner
        buf = torch.randn(n, device=dev)
        bufs = _register(L, ctx, buf, world)
        impls = {
            "p2p": lambda: L.hap_p2p_all_reduce(ctx, bufs.data_ptr(), bufs.data_ptr(), F32, n, cap, s),
            "nccl": lambda: L.hap_all_reduce(group.comm, buf.data_ptr(), buf.data_ptr(), n, F32, s),
        }
        for name, fn in impls.items():
            results.append({"op": "all_reduce", "impl": name, "rows": rows, "bytes": n * 4,
                            "s": timed(fn, f"all_reduce {name}")})
        # ---- all-to-all: [rows, inner] sharded by rows -> sharded by columns
        csz = round_shards(inner, ratios)
        send_counts = [sizes[rank] * c for c in csz]
        recv_counts = [sizes[j] * csz[rank] for j in range(world)]
        a2a_send = torch.randn(max(1, sum(send_counts)), device=dev).to(torch.bfloat16)
        a2a_recv = torch.empty(max(1, sum(recv_counts)), device=dev, dtype=torch.bfloat16)
        recvs = _register(L, ctx, a2a_recv, world)
        dst_off = [sum(sizes[i] * csz[k] for i in range(rank)) for k in range(world)]
        meta = torch.tensor([offsets(send_counts)[:-1], send_counts, dst_off], dtype=torch.int64, device=dev)
        sarr, rarr = i64_array(send_counts), i64_array(recv_counts)
        impls = {
            "p2p": lambda: L.hap_p2p_all_to_all(ctx, a2a_send.data_ptr(), recvs.data_ptr(), BF16, meta[0].data_ptr(),
                                                meta[1].data_ptr(), meta[2].data_ptr(), max(send_counts), cap, s),
            "nccl": lambda: L.hap_all_to_all_v(group.comm, a2a_send.data_ptr(), sarr, a2a_recv.data_ptr(), rarr, BF16,
                                               s),
        }
        # expected receive buffer from every rank's send buffer (host)
        sends = [None] * world
        dist.all_gather_object(sends, a2a_send.float().cpu())
        want = []
        for j in range(world):
            sc = [sizes[j] * c for c in csz]
            o = sum(sc[:rank])
            want.append(sends[j][o:o + sc[rank]])
        want = torch.cat(want)
        for name, fn in impls.items():
            # cleared and visible on every rank before any rank's kernel may
            # push into it (the zeroing runs on another stream than the call)
            torch.cuda.synchronize(dev)
            a2a_recv.zero_()
            torch.cuda.synchronize(dev)
            dist.barrier()
            check(fn(), name)
            torch.cuda.synchronize(dev)
            got = a2a_recv.float().cpu()[:want.numel()]
            if not torch.equal(got, want):
                bad = (got != want).nonzero().flatten()
                print(f"[rank {rank}] all_to_all {name} rows {rows}: {bad.numel()} of {want.numel()} elements wrong, "
                      f"first at {int(bad[0])}", flush=True)
                results.append({"op": "all_to_all", "impl": name, "rows": rows, "mismatch": int(bad.numel())})
            results.append({"op": "all_to_all", "impl": name, "rows": rows, "bytes": total_b16,
                            "s": timed(fn, f"all_to_all {name}")})
        if rank == 0:
            line = "  ".join(f"{r['op']}/{r['impl']} {r['s'] * 1e6:8.1f}us" for r in results[-8:] if "s" in r)
            print(f"rows {rows:7d} ({total_b16 / 1e6:8.3f} MB): {line}", flush=True)
    if rank == 0 and args.json:
        with open(args.json, "w") as fh:
            json.dump({"world": world, "caps": caps, "inner": inner, "results": results}, fh, indent=1)
    dist.barrier()
    check(L.hap_symm_destroy(ctx))
    group.close()
    dist.destroy_process_group()


def fit(paths, out):
    from paper_2401_05965_b200.cost_model import fit_linear

    model = {}
    if os.path.exists(out):   # keep the other world sizes' lines
        with open(out) as fh:
            model = json.load(fh)
    for path in paths:
        with open(path) as fh:
            doc = json.load(fh)
        world = str(doc["world"])
        model[world] = {}
        for op in OPS:
            for impl in ("p2p", "nccl"):
                samples = [(r["bytes"], r["s"]) for r in doc["results"]
                           if r["op"] == op and r["impl"] == impl and "s" in r]
                if len(samples) < 2:
                    continue
                f = fit_linear(samples)
                model.setdefault(world, {}).setdefault(op, {})[impl] = {
                    "latency_s": max(f.latency_s, min(t for _, t in samples) * 0.5),
                    "bw_Bps": f.bytes_per_second, "residual_s": f.residual,
                    "samples": [[b, t] for b, t in samples]}
    with open(out, "w") as fh:
        json.dump(model, fh, indent=1, sort_keys=True)
        fh.write("\n")
    for world, ops in sorted(model.items()):
        for op, impls in ops.items():
            print(world, op, {k: (round(v["latency_s"] * 1e6, 2), round(v["bw_Bps"] / 1e9, 1)) for k, v in impls.items()})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rows", default="16,64,256,1024,4096,16384,65536")
    ap.add_argument("--fit", nargs="*", default=None, help="fit the given sweep files instead of measuring")
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2401_05965_b200", "collectives_b200.json"))
    args = ap.parse_args()
    if args.fit:
        fit(args.fit, args.out)
    else:
        bench(args)


if __name__ == "__main__":
    main()
