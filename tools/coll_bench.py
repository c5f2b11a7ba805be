"""Uneven all-gather / reduce-scatter bandwidth: NVLink peer-memory kernel vs
NCCL (padded all-gather, grouped send/recv), shards weighted by the bench's
SM-cap ratios.  Run with torchrun (one process per GPU):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/coll_bench.py [--json out]

Reports, per implementation and size, the time (max over ranks, CUDA events)
and the bus bandwidth = bytes each rank must receive / time.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2401_05965_b200 import workloads  # noqa: E402
from paper_2401_05965_b200._lib import BF16, check, i64_array, lib  # noqa: E402
from paper_2401_05965_b200.executor import NcclGroup  # noqa: E402
from paper_2401_05965_b200.sharding import offsets, round_shards  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rows", default="4096,16384,65536,262144", help="comma-separated gathered row counts")
    ap.add_argument("--rs-rows", default="16384,65536,262144", help="comma-separated reduce-scatter row counts")
    ap.add_argument("--probe", default="", help="comma-separated MB per peer for the push/pull bandwidth probe")
    ap.add_argument("--ar-elems", default="", help="comma-separated fp32 all-reduce sizes (elements)")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    L = lib()
    group = NcclGroup.from_torch_distributed()
    caps = workloads.sm_caps(world)
    ratios = [c / sum(caps) for c in caps]
    inner = 768
    stream = torch.cuda.Stream(dev)
    results = []
    import ctypes
    arena_bytes = 1 << 30
    ctx = ctypes.c_void_p()
    check(L.hap_symm_create(ctypes.byref(ctx), arena_bytes, rank, world))
    h = ctypes.create_string_buffer(64)
    check(L.hap_symm_handle(ctx, h))
    handles = [None] * world
    dist.all_gather_object(handles, bytes(h.raw))
    check(L.hap_symm_open(ctx, b"".join(handles)))
    for rows in [int(v) for v in args.rows.split(",")]:
        sizes = round_shards(rows, ratios)
        counts = [s * inner for s in sizes]
        send = torch.randn(counts[rank], device=dev).to(torch.bfloat16)
        out = torch.empty(rows * inner, device=dev, dtype=torch.bfloat16)
        scratch = torch.empty(world * max(counts), device=dev, dtype=torch.bfloat16)
        devsz = torch.tensor([sizes, offsets(sizes)[:-1]], dtype=torch.int64, device=dev)
        carr = i64_array(counts)
        recv_bytes = (sum(counts) - counts[rank]) * 2
        # register `out` for the push kernel (the executor does this once per gather at compile time)
        hb = ctypes.create_string_buffer(64)
        base, boff = ctypes.c_int64(), ctypes.c_int64()
        check(L.hap_p2p_buffer_handle(ctx, out.data_ptr(), hb, ctypes.byref(base), ctypes.byref(boff)))
        trip = [None] * world
        dist.all_gather_object(trip, (bytes(hb.raw), base.value, boff.value))
        ptrs = (ctypes.c_void_p * world)()
        check(L.hap_p2p_buffer_open(ctx, out.data_ptr(), b"".join(t[0] for t in trip), i64_array([t[1] for t in trip]),
                                    i64_array([t[2] for t in trip]), ptrs))
        dev_outs = torch.tensor([int(p or 0) for p in ptrs], dtype=torch.int64, device=dev)
        impls = {
            "p2p_kernel": lambda: L.hap_p2p_all_gather_v(ctx, send.data_ptr(), out.data_ptr(), BF16, 1, inner, rows,
                                                         devsz[0].data_ptr(), devsz[1].data_ptr(), max(counts), 0,
                                                         stream.cuda_stream),
            "nccl_padded": lambda: L.hap_all_gather_v(group.comm, send.data_ptr(), out.data_ptr(), carr, BF16, 1,
                                                      scratch.data_ptr(), stream.cuda_stream),
            "nccl_sendrecv": lambda: L.hap_all_gather_v(group.comm, send.data_ptr(), out.data_ptr(), carr, BF16, 0,
                                                        None, stream.cuda_stream),
            "p2p_push": lambda: L.hap_p2p_all_gather_push(ctx, send.data_ptr(), dev_outs.data_ptr(), BF16, 1, inner,
                                                          rows, devsz[0].data_ptr(), devsz[1].data_ptr(), rows * inner,
                                                          0, stream.cuda_stream),
        }
        ref = None
        for name, fn in impls.items():
            out.zero_()   # each implementation must produce the whole output itself
            for _ in range(3):
                check(fn(), name)
            torch.cuda.synchronize(dev)
            if ref is None:
                ref = out.clone()
            else:
                assert torch.equal(out, ref), name
            dist.barrier()
            # 10 calls per CUDA graph: device time per call, no host launch cost
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
                for _ in range(10):
                    fn()
            torch.cuda.synchronize(dev)
            dist.barrier()
            with torch.cuda.stream(stream):
                graph.replay()
            torch.cuda.synchronize(dev)
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, args.reps // 10)
            e0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(reps):
                    graph.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            del graph
            t = torch.tensor([e0.elapsed_time(e1) / (reps * 10)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            rb = torch.tensor([recv_bytes], device=dev, dtype=torch.float64)
            dist.all_reduce(rb, op=dist.ReduceOp.MAX)
            # NVLink-bound bytes at the measured 770 GB/s per direction: every
            # rank receives all other shards (ingress) and its shard leaves it
            # m-1 times (egress — pushed, or read by the peers); the padded
            # NCCL gather moves the largest shard's size from every rank
            b = 2 * inner
            ingress = (sum(sizes) - min(sizes)) * b
            egress = (world - 1) * max(sizes) * b
            bound = (world - 1) * max(sizes) * b if name == "nccl_padded" else max(ingress, egress)
            results.append({"op": "all_gather", "impl": name, "rows": rows, "shard_rows": sizes,
                            "ms": ms, "recv_GBps_max_rank": float(rb.item()) / (ms * 1e-3) / 1e9,
                            "nvlink_bound_bytes": bound,
                            "frac_of_770": bound / (ms * 1e-3) / 770e9})
    # uneven reduce-scatter: staged pull kernel, direct kernel on registered partials, NCCL
    for rows in [int(v) for v in args.rs_rows.split(",") if v]:
        sizes = round_shards(rows, ratios)
        counts = [sz * inner for sz in sizes]
        send = torch.randn(rows * inner, device=dev).to(torch.bfloat16)
        out = torch.empty(counts[rank], device=dev, dtype=torch.bfloat16)
        scratch = torch.empty(world * max(counts), device=dev, dtype=torch.bfloat16)
        devsz = torch.tensor([sizes, offsets(sizes)[:-1]], dtype=torch.int64, device=dev)
        carr = i64_array(counts)
        hb = ctypes.create_string_buffer(64)
        base, boff = ctypes.c_int64(), ctypes.c_int64()
        check(L.hap_p2p_buffer_handle(ctx, send.data_ptr(), hb, ctypes.byref(base), ctypes.byref(boff)))
        trip = [None] * world
        dist.all_gather_object(trip, (bytes(hb.raw), base.value, boff.value))
        ptrs = (ctypes.c_void_p * world)()
        check(L.hap_p2p_buffer_open(ctx, send.data_ptr(), b"".join(t[0] for t in trip),
                                    i64_array([t[1] for t in trip]), i64_array([t[2] for t in trip]), ptrs))
        dev_sends = torch.tensor([int(p or 0) for p in ptrs], dtype=torch.int64, device=dev)
        impls = {
            "p2p_rs_staged": lambda: L.hap_p2p_reduce_scatter_v(ctx, send.data_ptr(), out.data_ptr(), BF16, 1, inner,
                                                                rows, devsz[0].data_ptr(), devsz[1].data_ptr(), 0,
                                                                stream.cuda_stream),
            "p2p_rs_direct": lambda: L.hap_p2p_reduce_scatter_direct(ctx, dev_sends.data_ptr(), out.data_ptr(), BF16,
                                                                     1, inner, rows, devsz[0].data_ptr(),
                                                                     devsz[1].data_ptr(), counts[rank], 0,
                                                                     stream.cuda_stream),
            "nccl_rs": lambda: L.hap_reduce_scatter_v(group.comm, send.data_ptr(), out.data_ptr(), carr, BF16,
                                                      scratch.data_ptr(), stream.cuda_stream),
        }
        ref = None
        for name, fn in impls.items():
            out.zero_()
            for _ in range(3):
                check(fn(), name)
            torch.cuda.synchronize(dev)
            if ref is None:
                ref = out.clone()
            elif name.startswith("p2p"):
                assert torch.equal(out, ref), name   # same fp32 sum order, one rounding
            diff = float((out.float() - ref.float()).abs().max())   # NCCL: bf16 partial sums
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
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, args.reps // 10)
            e0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(reps):
                    graph.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            del graph
            t = torch.tensor([e0.elapsed_time(e1) / (reps * 10)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            b = 2 * inner
            # rank j reads its rows from m-1 peers (ingress (m-1) size_j); its
            # partial's other rows leave it (egress rows - size_j)
            ingress = (world - 1) * max(sizes) * b
            egress = (rows - min(sizes)) * b
            bound = max(ingress, egress)
            results.append({"op": "reduce_scatter", "impl": name, "rows": rows, "shard_rows": sizes, "ms": ms,
                            "max_abs_diff_vs_p2p": diff,
                            "recv_GBps_max_rank": ingress / (ms * 1e-3) / 1e9, "nvlink_bound_bytes": bound,
                            "frac_of_770": bound / (ms * 1e-3) / 770e9})
    # raw NVLink bandwidth: pull vs push, peers in turn vs all at once
    for mb in [int(v) for v in args.probe.split(",") if v]:
        chunk = mb << 20
        for mode, name in enumerate(["pull_seq", "push_seq", "pull_split", "push_split", "local_copy"]):
            fn = lambda: L.hap_p2p_probe(ctx, mode, chunk, 0, stream.cuda_stream)  # noqa: E731
            check(fn(), name)
            torch.cuda.synchronize(dev)
            ts = []
            for _ in range(5):
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                check(fn(), name)
                e1.record(stream)
                torch.cuda.synchronize(dev)
                ts.append(e0.elapsed_time(e1))
            t = torch.tensor([sorted(ts)[len(ts) // 2]], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            results.append({"op": "probe", "impl": name, "rows": mb, "shard_rows": [], "ms": ms,
                            "recv_GBps_max_rank": (world - 1) * chunk / (ms * 1e-3) / 1e9})
    # NCCL all-reduce (fp32, in place) — the gradient synchronisation
    for elems in [int(v) for v in args.ar_elems.split(",") if v]:
        buf = torch.randn(elems, device=dev)
        fn = lambda: L.hap_all_reduce(group.comm, buf.data_ptr(), buf.data_ptr(), elems, 0,  # noqa: E731
                                      stream.cuda_stream)
        for _ in range(3):
            check(fn(), "all_reduce")
        torch.cuda.synchronize(dev)
        dist.barrier()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
            for _ in range(10):
                fn()
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, args.reps // 10)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(reps):
                graph.replay()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        del graph
        t = torch.tensor([e0.elapsed_time(e1) / (reps * 10)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        # bus bandwidth convention: 2 (n-1)/n x bytes / time
        results.append({"op": "all_reduce", "impl": "nccl", "rows": elems, "shard_rows": [],
                        "ms": ms, "recv_GBps_max_rank": 2 * (world - 1) / world * elems * 4 / (ms * 1e-3) / 1e9})
    if rank == 0:
        for r in results:
            print(f"{r['op']:10s} {r['impl']:14s} rows={r['rows']:7d} {r['ms'] * 1e3:9.1f} us "
                  f"{r['recv_GBps_max_rank']:7.1f} GB/s received per rank"
                  + (f"  {100 * r['frac_of_770']:5.1f}% of 770 GB/s on the bound direction" if "frac_of_770" in r else ""))
        if args.json:
            with open(args.json, "w") as fh:
                json.dump({"world": world, "caps": caps, "results": results}, fh, indent=1)
    dist.barrier()
    check(L.hap_symm_destroy(ctx))
    group.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
