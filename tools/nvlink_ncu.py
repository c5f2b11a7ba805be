"""NVLink traffic of the peer-memory collectives, for an ncu capture of the
NVLRX / NVLTX byte counters (one pass: no kernel replay, so the kernels'
cross-GPU flag waits are safe under the profiler):

    ncu --target-processes all -k regex:p2p_ --clock-control none --csv \\
        --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,\\
nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \\
        --log-file gpurun_out/nvl.csv \\
        torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_ncu.py

--nvml (no profiler): the GPU's NVLink data counters (NVML field values
NVLINK_THROUGHPUT_DATA_TX / _RX, summed over the links, KiB) are read before
and after `--reps` back-to-back calls of each collective; the line then holds
the counted NVLink bytes per call beside the algorithmic ones and the
achieved GB/s from CUDA events over the same calls (max over ranks).

Each rank runs, eagerly with a barrier between calls, the push all-gather,
the direct reduce-scatter, the two-shot all-reduce and the push all-to-all of
a [rows, 768] bf16 tensor sharded by the bench's SM-cap ratios (the executor's
buffers, registered the same way), and prints the algorithmic bytes each rank
must receive / send per call so the counters can be set against them
(tools/summarize_nvlink.py).  Without ncu it prints CUDA-event times.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def _nvlink_kib(index: int) -> tuple[int, int]:
    """(tx, rx) NVLink data KiB of GPU `index` since boot, summed over its links."""
    import pynvml as nv

    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(index)
    tx = rx = 0
    for link in range(18):
        try:
            vals = nv.nvmlDeviceGetFieldValues(h, [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                                                   (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
        except nv.NVMLError:
            break
        if vals[0].nvmlReturn or vals[1].nvmlReturn:
            continue
        tx += vals[0].value.ullVal
        rx += vals[1].value.ullVal
    return tx, rx


class _Gpm:
    """NVLink RX / TX of one GPU between two GPM samples (NVML GPU
    Performance Monitoring: NVLINK_TOTAL_RX/TX_PER_SEC, MiB/s averaged over the
    interval between the samples, all links)."""

    def __init__(self, index: int):
        import pynvml as nv

        nv.nvmlInit()
        self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(index)
        self.ok = bool(nv.nvmlGpmQueryDeviceSupport(self.h).isSupportedDevice)
        self.s1, self.s2 = nv.nvmlGpmSampleAlloc(), nv.nvmlGpmSampleAlloc()

    def start(self):
        import time

        self.nv.nvmlGpmSampleGet(self.h, self.s1)
        self.t0 = time.perf_counter()

    def stop(self) -> tuple[float, float]:
        """(tx, rx) bytes moved over NVLink since start()."""
        import time

        self.nv.nvmlGpmSampleGet(self.h, self.s2)
        dt = time.perf_counter() - self.t0
        nv = self.nv
        mg = nv.c_nvmlGpmMetricsGet_t()
        mg.version = nv.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 2
        mg.sample1, mg.sample2 = self.s1, self.s2
        mg.metrics[0].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
        mg.metrics[1].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
        nv.nvmlGpmMetricsGet(mg)
        return mg.metrics[0].value * (1 << 20) * dt, mg.metrics[1].value * (1 << 20) * dt


def main():
    import torch
    import torch.distributed as dist

    from coll_fit import _register
    from paper_2401_05965_b200 import workloads
    from paper_2401_05965_b200._lib import BF16, check, lib
    from paper_2401_05965_b200.sharding import offsets, round_shards

    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="16384,65536")
    ap.add_argument("--calls", type=int, default=3)
    ap.add_argument("--json", default=None)
    ap.add_argument("--nvml", action="store_true", help="NVML NVLink byte counters instead of an ncu capture")
    ap.add_argument("--reps", type=int, default=100)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    L = lib()
    caps = workloads.sm_caps(world)
    cap = caps[rank]
    ratios = [c / sum(caps) for c in caps]
    inner = 768
    ctx = ctypes.c_void_p()
    check(L.hap_symm_create(ctypes.byref(ctx), 1 << 20, rank, world))
    h = ctypes.create_string_buffer(64)
    check(L.hap_symm_handle(ctx, h))
    handles = [None] * world
    dist.all_gather_object(handles, bytes(h.raw))
    check(L.hap_symm_open(ctx, b"".join(handles)))
    stream = torch.cuda.current_stream(dev).cuda_stream
    report = []
    gpm = None
    if args.nvml:
        try:
            gpm = _Gpm(local)
            if not gpm.ok:
                gpm = None
        except Exception as exc:  # noqa: BLE001 - fall back to the field counters
            print(f"[rank {rank}] GPM unavailable: {exc}", flush=True)
    for rows in [int(v) for v in args.rows.split(",")]:
        sizes = round_shards(rows, ratios)
        offs = offsets(sizes)
        counts = [sz * inner for sz in sizes]
        devsz = torch.tensor([sizes, offs[:-1]], dtype=torch.int64, device=dev)
        send = torch.randn(max(1, counts[rank]), device=dev).to(torch.bfloat16)
        out = torch.empty(rows * inner, device=dev, dtype=torch.bfloat16)
        outs = _register(L, ctx, out, world)
        part = torch.randn(rows * inner, device=dev).to(torch.bfloat16)
        parts = _register(L, ctx, part, world)
        rs_out = torch.empty(max(1, counts[rank]), device=dev, dtype=torch.bfloat16)
        ar = torch.randn(rows * inner, device=dev).to(torch.bfloat16)
        ars = _register(L, ctx, ar, world)
        csz = round_shards(inner, ratios)
        send_counts = [sizes[rank] * c for c in csz]
        recv_counts = [sizes[j] * csz[rank] for j in range(world)]
        a2a_send = torch.randn(max(1, sum(send_counts)), device=dev).to(torch.bfloat16)
        a2a_recv = torch.empty(max(1, sum(recv_counts)), device=dev, dtype=torch.bfloat16)
        recvs = _register(L, ctx, a2a_recv, world)
        dst_off = [sum(sizes[i] * csz[k] for i in range(rank)) for k in range(world)]
        meta = torch.tensor([offsets(send_counts)[:-1], send_counts, dst_off], dtype=torch.int64, device=dev)
        b = 2
        ops = {
            # name: (call, bytes received per rank, bytes sent per rank)
            "all_gather_push": (lambda: L.hap_p2p_all_gather_push(ctx, send.data_ptr(), outs.data_ptr(), BF16, 1,
                                                                  inner, rows, devsz[0].data_ptr(),
                                                                  devsz[1].data_ptr(), rows * inner, cap, stream),
                                (rows - sizes[rank]) * inner * b, (world - 1) * sizes[rank] * inner * b),
            "reduce_scatter_direct": (lambda: L.hap_p2p_reduce_scatter_direct(ctx, parts.data_ptr(), rs_out.data_ptr(),
                                                                              BF16, 1, inner, rows, devsz[0].data_ptr(),
                                                                              devsz[1].data_ptr(), counts[rank], cap,
                                                                              stream),
                                      (world - 1) * sizes[rank] * inner * b, (rows - sizes[rank]) * inner * b),
            "all_reduce": (lambda: L.hap_p2p_all_reduce(ctx, ars.data_ptr(), ars.data_ptr(), BF16, rows * inner, cap,
                                                        stream),
                           2 * (world - 1) * rows * inner * b // world, 2 * (world - 1) * rows * inner * b // world),
            "all_to_all_push": (lambda: L.hap_p2p_all_to_all(ctx, a2a_send.data_ptr(), recvs.data_ptr(), BF16,
                                                             meta[0].data_ptr(), meta[1].data_ptr(), meta[2].data_ptr(),
                                                             max(send_counts), cap, stream),
                                (sum(recv_counts) - recv_counts[rank]) * b, (sum(send_counts) - send_counts[rank]) * b),
        }
        if args.nvml:
            for name, (fn, rx, tx) in ops.items():
                check(fn(), name)
                torch.cuda.synchronize(dev)
                dist.barrier()
                c0 = _nvlink_kib(local)
                if gpm is not None:
                    try:
                        gpm.start()
                    except Exception as exc:  # noqa: BLE001 - GPM sampling refused on this box
                        print(f"[rank {rank}] GPM sampling failed ({exc}); NVML field counters only", flush=True)
                        gpm = None
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.reps):
                    check(fn(), name)
                e1.record()
                torch.cuda.synchronize(dev)
                g_tx, g_rx = gpm.stop() if gpm is not None else (0.0, 0.0)
                c1 = _nvlink_kib(local)
                ms = torch.tensor([e0.elapsed_time(e1) / args.reps], device=dev)
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
                t = float(ms) * 1e-3
                ctx_b = (c1[0] - c0[0]) * 1024 / args.reps, (c1[1] - c0[1]) * 1024 / args.reps
                if ctx_b == (0, 0) and (g_tx or g_rx):   # field counters not reported: GPM rates x interval
                    ctx_b = g_tx / args.reps, g_rx / args.reps
                report.append({"rank": rank, "op": name, "rows": rows, "rx_bytes": rx, "tx_bytes": tx,
                               "us_per_call_max_over_ranks": round(t * 1e6, 2),
                               "nvlink_tx_bytes_counted": ctx_b[0], "nvlink_rx_bytes_counted": ctx_b[1],
                               "alg_GBps": round(max(rx, tx) / t / 1e9, 1),
                               "counted_GBps": round(max(ctx_b) / t / 1e9, 1),
                               "frac_of_770": round(max(rx, tx) / t / 770e9, 3)})
            continue
        for name, (fn, rx, tx) in ops.items():
            times = []
            for _ in range(args.calls):
                dist.barrier()
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                check(fn(), name)
                e1.record()
                torch.cuda.synchronize(dev)
                times.append(e0.elapsed_time(e1))
            report.append({"rank": rank, "op": name, "rows": rows, "rx_bytes": rx, "tx_bytes": tx,
                           "event_ms_min": min(times)})
    everyone = [None] * world
    dist.all_gather_object(everyone, report)
    if rank == 0:
        flat = [r for sub in everyone for r in sub]
        for r in flat:
            print(json.dumps(r))
        if args.json:
            with open(args.json, "w") as fh:
                json.dump({"world": world, "caps": caps, "calls": args.calls, "rows": args.rows, "ranks": flat}, fh,
                          indent=1)
    dist.barrier()
    check(L.hap_symm_destroy(ctx))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
