"""Benchmark: training iterations of a HAP-synthesized program on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[2]): the BERT-base GEMM skeleton (12 layers,
seq 128, hidden 768, FFN 3072) in the reference IR, 64 sequences per GPU
(global batch 64*N, weak scaling), planned by HAP for N devices whose speeds
are per-rank SM caps (148/104/132/88 SMs: heterogeneity emulated on the
homogeneous box), executed by the B200 executor: one process per GPU, NCCL
collectives, tcgen05 GEMMs, every kernel grid capped at the rank's SMs.  One
step = forward + adjoint backward + gradient sync (all-reduce or SFB, cost
model) + SGD update, replayed as one CUDA graph.

``--workload moe`` runs configs[4] instead: a 12-layer stack of 2-expert SiLU
FFN mixtures at 2 sequences per GPU, where the cost model picks sufficient-
factor broadcasting (gather x and dy, rebuild dW locally) at 2 and 4 GPUs and
all-reduce at 8 (the grad_sync map in ``config`` records each choice).

The printed JSON line follows the driver contract; ``value`` is samples
(sequences) per second for the whole job with inputs resident in HBM,
``e2e`` the same metric through the public API with the batch copied from
pinned host memory and the loss read back every step.
"""
from __future__ import annotations

import argparse
import json
import math
import os

# one hardware work queue per stream (see paper_2401_05965_b200/__init__.py);
# must precede CUDA context creation
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEQ = 128
LAYERS = 12
# --workload: graph builder, sequences per GPU, plan-file stem, description.
WORKLOADS = {
    "bert": {"per_gpu_batch": 64, "stem": "bert12",
             "desc": "BERT-base GEMM skeleton (configs[2]): 12 layers, seq 128, hidden 768, FFN 3072, "
                     "train step fwd+bwd+sync+SGD"},
    "moe": {"per_gpu_batch": 2, "stem": "moe12",
            "desc": "BERT-MoE FFN stack (configs[4]): 12 layers x 2 SiLU experts (768->3072->768), seq 128, "
                    "SFB-vs-all-reduce chosen per weight by the cost model, train step fwd+bwd+sync+SGD"},
    "vitmoe": {"per_gpu_batch": 16, "stem": "vitmoe12", "seq": 197,
               "desc": "ViT-MoE skeleton (configs[3]): 12 ViT-B/16 blocks (197 tokens, hidden 768), each an "
                       "attention skeleton + 2 SiLU experts (768->3072->768) expert-sliced over the GPUs: uneven "
                       "all-gather / reduce-scatter per layer (program from the reference's program space, LP "
                       "ratios), train step fwd+bwd+sync+SGD"},
}


def _seq(workload: str) -> int:
    return WORKLOADS[workload].get("seq", SEQ)


def _graph(workload: str, batch: int):
    from paper_2401_05965_b200 import workloads
    if workload == "vitmoe":
        return workloads.vit_moe(layers=LAYERS, experts=2, images=batch, tokens=_seq(workload))
    if workload == "moe":
        return workloads.moe_stack(layers=LAYERS, batch=batch, seq=SEQ)
    return workloads.bert(layers=LAYERS, batch=batch, seq=SEQ)
# SGD step size.  The skeleton's loss is the reference's plain sum over
# batch*seq*768 outputs (unbounded below, gradients ~1e4-1e5 per weight), so
# the step is chosen to move weights ~1e-5 relative per step: long runs stay
# finite.  The update kernel reads and writes every master/weight/gradient
# element regardless of the step size.
LR = 1e-11


def _peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            doc = json.load(fh)
        return {"hbm_gbs": doc["hbm_gbs"], "bf16_tflops": doc["bf16_tflops"],
                "bf16_tflops_sustained": doc.get("bf16_tflops_sustained", doc["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


def _plan_doc(workload: str, n: int) -> dict:
    """The reference planner's plan for n devices (tests/golden/plans, made by
    tests/golden/make_golden.py from the reference package).  N = 1 uses the
    N = 2 plan's program re-targeted to one device: the planner emits the
    same program at every device count (tests/test_workloads.py), but its
    m = 1 search does not finish at 12 layers (workloads.planned_program)."""
    w = WORKLOADS[workload]
    k = max(n, 2)
    path = os.path.join(ROOT, "tests", "golden", "plans", f"{w['stem']}_b{w['per_gpu_batch'] * k}.b200x{k}.json")
    with open(path) as fh:
        return json.load(fh)


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    An NVML polling thread (every 5 ms, plus one sample on entry and one on
    exit, so even a short timed region has samples); the nvidia-smi CSV loop
    of the profiling recipe is the fallback when NVML is unavailable.  The
    device is addressed by PCI bus id, so CUDA_VISIBLE_DEVICES remapping
    cannot point the sampler at another GPU."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.samples = []          # (sm_mhz, reasons)
        self.sm_max = None
        self._stop = None
        self._thread = None
        self._nvml = None
        self._handle = None
        self._smi = None

    def _sample(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._handle, nv.NVML_CLOCK_SM)
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._handle)
        self.samples.append((float(sm), {name for name, attr in self.REASONS if mask & getattr(nv, attr)}))

    def _loop(self):
        while not self._stop.wait(self.period):
            try:
                self._sample()
            except Exception:  # noqa: BLE001 - a failed sample is just missing
                pass

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            self._nvml = nv
            self._handle = nv.nvmlDeviceGetHandleByPciBusId(bus)
            self.sm_max = float(nv.nvmlDeviceGetMaxClockInfo(self._handle, nv.NVML_CLOCK_SM))
            self._sample()
            self._stop = threading.Event()
            self._thread = threading.Thread(target=self._loop, daemon=True)
            self._thread.start()
        except Exception:  # noqa: BLE001 - fall back to the nvidia-smi loop
            self._nvml = None
            try:
                self._smi = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.index}",
                     "--query-gpu=index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                     "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except OSError:
                self._smi = None
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join()
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                pass
        if self._smi is not None:
            self._smi.terminate()
            try:
                out, _ = self._smi.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self._smi.kill()
                out, _ = self._smi.communicate()
            for ln in out.splitlines():
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm, smax = float(parts[1]), float(parts[2])
                except ValueError:
                    continue
                self.sm_max = max(self.sm_max or 0.0, smax)
                self.samples.append((sm, {name for (name, _), flag in zip(self.REASONS, parts[3:7])
                                          if flag.lower() == "active"}))

    def summary(self) -> dict:
        sm = [s for s, _ in self.samples]
        reasons = set().union(*[r for _, r in self.samples]) if self.samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.sm_max,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def cpu_baseline(steps: int, sample_batch: int, workload: str = "bert", budget_s: float = 30.0) -> dict:
    """Reference CPU path (the oracle port of the reference interpreter plus
    its adjoint, float64 numpy) on a bounded sample of the same workload:
    up to ``steps`` train steps, stopping once ``budget_s`` seconds of CPU
    work are measured, with every host core given to the BLAS pool (torchrun
    sets OMP_NUM_THREADS=1 per rank)."""
    import numpy as np  # noqa: F401
    from threadpoolctl import threadpool_info, threadpool_limits

    from oracle import interpreter_np as O
    from paper_2401_05965_b200 import workloads

    threadpool_limits(limits=os.cpu_count() or 1)
    g = _graph(workload, sample_batch)
    planned, table, _ = workloads.planned_program(g, 1, _plan_doc(workload, 1))
    prog = O.Program(planned.to_json())
    inputs = workloads.synthetic_inputs(g, 0, scaled=True)
    shapes = {n.id: n.shape for n in g.nodes}
    O.train_step(prog, 1, inputs, table, shapes, lr=1e-3)  # warm
    t0 = time.perf_counter()
    done = 0
    while done < max(1, steps):
        O.train_step(prog, 1, inputs, table, shapes, lr=1e-3)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    steps = done
    dt = (time.perf_counter() - t0) / steps
    threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    return {"value": sample_batch / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{steps} train steps (fwd+bwd+SGD, float64) of the planner's 12-layer {workload} program "
                      f"at batch {sample_batch} x seq {_seq(workload)} on one simulated device",
            "seconds_per_step": dt}


def run_reference_arm(args, rank: int) -> None:
    if rank != 0:
        return
    sample = 4 if args.workload == "bert" else 2
    cb = cpu_baseline(max(1, args.steps), sample_batch=sample, workload=args.workload)
    line = {"impl": "reference", "metric": "samples/sec per train iter of HAP program", "value": cb["value"],
            "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.workload]["desc"],
                       "global_batch": sample, "seq_len": _seq(args.workload), "parallelism": "cpu"},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit_json(line)


# stdout carries exactly one JSON line: libraries that print to fd 1 (NCCL's
# version banner at communicator init) are pointed at stderr, and the
# result is written to the saved original stdout.
_STDOUT_FD = None


def _quiet_stdout():
    global _STDOUT_FD
    if _STDOUT_FD is None:
        sys.stdout.flush()
        _STDOUT_FD = os.dup(1)
        os.dup2(2, 1)


def emit_json(line: dict) -> None:
    data = (json.dumps(line) + "\n").encode()
    if _STDOUT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        sys.stdout.flush()
        os.write(_STDOUT_FD, data)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="bert", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch ops eagerly instead of one CUDA graph")
    ap.add_argument("--grad-sync", default="auto", choices=["auto", "sfb", "all_reduce"],
                    help="replicated-weight gradient sync: the cost model's pick per weight, or forced")
    ap.add_argument("--collectives", default="auto", choices=["auto", "p2p", "nccl"],
                    help="auto: NCCL group, kernel or NCCL per call site; p2p: NVLink peer-memory kernels only "
                         "(no NCCL communicator); nccl: NCCL only")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2401_05965_b200 import _lib, workloads
    from paper_2401_05965_b200.cost_model import ClusterSpec
    from paper_2401_05965_b200.executor import ExecConfig, Executor, LocalGroup, NcclGroup, PeerGroup
    from paper_2401_05965_b200.program import DistributedProgram
    from paper_2401_05965_b200.sharding import offsets, table_from_plan

    t_start = time.time()

    def log(msg):
        if args.verbose:
            print(f"[rank {rank} {time.time() - t_start:7.2f}s] {msg}", file=sys.stderr, flush=True)

    n = args.gpus
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    caps = workloads.sm_caps(n)
    cluster = ClusterSpec.from_dict(workloads.cluster_doc(caps))
    wl = WORKLOADS[args.workload]
    batch = wl["per_gpu_batch"] * n
    g = _graph(args.workload, batch)
    doc = _plan_doc(args.workload, n)
    if n == 1:
        prog, table, ratios = workloads.planned_program(g, 1, doc)
        plan_name = f"{wl['stem']}_b{wl['per_gpu_batch'] * 2}.b200x2 program on one device (planner's m=1 program)"
    else:
        prog, table = DistributedProgram.from_json(doc["program"]), table_from_plan(doc)
        ratios, plan_name = tuple(doc["ratios"][0]), f"{wl['stem']}_b{batch}.b200x{n}"
    if world == 1:
        group = LocalGroup(1)
    elif args.collectives == "p2p":
        group = PeerGroup.from_torch_distributed()
    else:
        group = NcclGroup.from_torch_distributed()
    gather = {"auto": "auto", "p2p": "kernel", "nccl": "sendrecv"}[args.collectives]
    shapes = {nd.id: nd.shape for nd in g.sources()}
    ex = Executor(prog, n, table, shapes, group=group,
                  config=ExecConfig(dtype="bf16", sm_caps=caps, lr=LR, cluster=cluster, ratios=ratios,
                                    grad_sync=args.grad_sync, gather=gather),
                  device=dev)
    log(f"executor compiled: {len(ex.ops_fwd)} fwd / {len(ex.ops_bwd)} bwd / {len(ex.ops_upd)} update ops; "
        f"weight-gradient GEMMs on the side stream (moved, forks, joins): {ex.wgrad_stats}")
    inputs = workloads.synthetic_inputs(g, 0, scaled=True)
    ex.load(inputs)
    ex.forward()
    log(f"inputs loaded, initial loss {ex.losses()[0]}")
    if not args.no_graph:
        ex.capture()
        log("graph captured")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        ex.step()
    barrier()
    log(f"warm, loss {ex.losses()[0]}")
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.profiler.start()   # `ncu --profile-from-start off` sees the timed steps only
        start.record(ex.stream)
        for _ in range(args.steps):
            ex.step()
        stop.record(ex.stream)
        barrier()
        torch.cuda.profiler.stop()
    ms_local = start.elapsed_time(stop)
    ms = torch.tensor([ms_local], device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(ms.item()) / args.steps
    losses = ex.losses()
    log(f"timed: {ms_per_step:.3f} ms/step, loss {losses[0]}")

    # ---- e2e through the public API: batch from pinned host memory, loss read back
    x0 = [ins for ins in prog.instrs if ins.ref == "x0" and ins.kind.startswith("placeholder")][0]
    host = torch.from_numpy(inputs["x0"].astype(np.float32)).to(torch.bfloat16).pin_memory()
    if x0.kind == "placeholder_shard":
        sizes = table[("x0", x0.axis)]
        lo, cnt = offsets(sizes)[group.rank], sizes[group.rank]
        host_part = host.narrow(x0.axis, lo, cnt)
        if x0.axis != 0:
            host_part = host_part.contiguous()
    else:
        host_part = host
    dst = ex.bufs[(x0.output, group.rank)].tensor[:host_part.numel()]
    # A prefetching input pipeline, as a data loader drives the executor:
    # step i+1's batch is copied host -> device (pinned, copy stream) into one
    # of two staging buffers while step i computes; each step starts with a
    # device copy staging -> the program's input buffer, and its loss is
    # copied back asynchronously and read on the host one step later (every
    # step's input and result still cross PCIe inside the timed region).
    src = host_part.reshape(-1)
    copy_stream = torch.cuda.Stream(dev)
    stage = [torch.empty_like(dst) for _ in range(2)]
    loss_host = torch.empty(max(1, args.steps), dtype=torch.float32).pin_memory()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_loss = [torch.cuda.Event() for _ in range(max(1, args.steps))]
    e2e_start, e2e_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def prefetch(i):
        slot = i % 2
        if i >= 2:   # the slot's previous batch has been copied into the program's input
            copy_stream.wait_event(ev_free[slot])
        with torch.cuda.stream(copy_stream):
            stage[slot].copy_(src, non_blocking=True)
            ev_in[slot].record(copy_stream)

    barrier()
    e2e_start.record(ex.stream)
    copy_stream.wait_event(e2e_start)
    prefetch(0)
    for i in range(args.steps):
        if i + 1 < args.steps:
            prefetch(i + 1)
        slot = i % 2
        ex.stream.wait_event(ev_in[slot])
        with torch.cuda.stream(ex.stream):
            dst.copy_(stage[slot], non_blocking=True)
            ev_free[slot].record(ex.stream)
        ex.step()
        with torch.cuda.stream(ex.stream):
            loss_host[i:i + 1].copy_(ex.loss_buf[group.rank].tensor[:1], non_blocking=True)
            ev_loss[i].record(ex.stream)
        if i > 0:
            ev_loss[i - 1].synchronize()
            _ = float(loss_host[i - 1])
    e2e_stop.record(ex.stream)
    ev_loss[args.steps - 1].synchronize()
    _ = float(loss_host[args.steps - 1])
    barrier()
    e2e_ms = torch.tensor([e2e_start.elapsed_time(e2e_stop) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    h2d = torch.tensor([host_part.numel() * 2], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(h2d)

    # ---- dominant kernel: the tcgen05 GEMMs of one step, replayed alone as one
    # CUDA graph on the executor stream (as inside the step: no host launch
    # cost between kernels), timed with CUDA events on that stream
    gemm_ops = [op for op in ex.ops_fwd + ex.ops_bwd if op.gemm is not None]
    reps = 10
    s_ptr = ex.stream.cuda_stream

    def launch_gemms():
        for op in gemm_ops:   # hap_matmul_batch(descs, count, sum_k, in_dt, out_dt, cap, stream)
            st = op.fn(*op.args[:-1], s_ptr)
            if st:
                _lib.check(st, op.what)

    gemm_graph = None
    try:
        launch_gemms()
        torch.cuda.synchronize(dev)
        gemm_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gemm_graph, stream=ex.stream):
            launch_gemms()
    except Exception as exc:  # noqa: BLE001 - eager replay as the fallback measurement
        log(f"GEMM graph capture failed ({exc}); timing eager launches")
        gemm_graph = None
    g_start, g_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    trials = []
    with ClockSampler(local) as gclk:
        for _ in range(3):   # best of three batches of `reps` replays
            g_start.record(ex.stream)
            with torch.cuda.stream(ex.stream):   # a graph replays on the current stream
                for _ in range(reps):
                    if gemm_graph is not None:
                        gemm_graph.replay()
                    else:
                        launch_gemms()
            g_stop.record(ex.stream)
            torch.cuda.synchronize(dev)
            trials.append(g_start.elapsed_time(g_stop) / reps)
    gemm_ms = min(trials)
    gemm_timing = "one CUDA graph of the step's GEMM launches" if gemm_graph is not None else "eager launches"
    gemm_graph = None
    members = [m for op in gemm_ops for m in op.gemm.get("members", [op.gemm])]
    gemm_flops = sum(2 * m["M"] * m["N"] * m["K"] for m in members)
    engines = {ex.lib.hap_matmul_engine(m["A"], m["lda"], m["transA"], m["B"], m["ldb"], m["transB"], m["M"],
                                        m["N"], m["K"], m["in_dt"]) for m in members}
    peaks = _peaks()
    achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12
    gemm_bytes = sum(2 * (m["M"] * m["K"] + m["K"] * m["N"]) + m["M"] * m["N"] * (2 if m["out_dt"] else 4)
                     * (2 if m["accumulate"] else 1) for m in members)
    traffic = None
    prof = next((q for q in (os.path.join(ROOT, "profiles", f"r{r}_gemm_traffic_{args.workload}.json")
                             for r in ("02", "01h")) if os.path.exists(q)), "")
    if n == 1 and prof:
        with open(prof) as fh:
            tr = json.load(fh)
        traffic = tr["dram_read_bytes_per_step"] + tr["dram_write_bytes_per_step"]
    # Binding resource at the algorithmic figures: the step's GEMMs are
    # tensor-bound when Σ flops / tensor peak exceeds Σ operand+output bytes /
    # HBM peak (BERT, 8192-token rows), HBM-bound otherwise (the MoE stack's
    # 256-token rows: the weights dominate, ~145 flop/B < the ~250 ridge).
    # Peak: the timed object is 3 x 10 replays of the step's GEMM launches
    # (tens of ms, not a seconds-long power-capped run), so the burst figure
    # of MEASURED_PEAKS.json is the denominator; the sustained one is beside it.
    t_tensor = gemm_flops / (peaks["bf16_tflops"] * 1e12)
    t_hbm = gemm_bytes / (peaks["hbm_gbs"] * 1e9)
    tensor_frac = achieved / peaks["bf16_tflops"]
    if t_hbm > t_tensor:
        gbs = gemm_bytes / (gemm_ms * 1e-3) / 1e9
        head = {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(gbs / peaks["hbm_gbs"], 4), "tensor_tflops": round(achieved, 1),
                "tensor_frac": round(tensor_frac, 4)}
    else:
        head = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": round(tensor_frac, 4)}
    roofline = {**head, "kernel": "gemm_tc2_kernel / gemm_tc_kernel (tcgen05, all GEMMs of one step)",
                "roofline_ms_per_step": round(max(t_tensor, t_hbm) * 1e3, 4),
                "peak_sustained": peaks["bf16_tflops_sustained"],
                "frac_sustained": round(achieved / peaks["bf16_tflops_sustained"], 4),
                "gemm_clocks": gclk.summary(), "traffic": traffic,
                "traffic_note": f"DRAM bytes per step over all GEMM launches (ncu, caches flushed per kernel; "
                                f"profiles/{os.path.basename(prof)})",
                "algorithmic_bytes_per_step": gemm_bytes, "gemm_flops_per_step": gemm_flops,
                "peak_source": peaks["source"] + ", burst (the GEMM replay is tens of ms); sustained in "
                               "peak_sustained",
                "timing": gemm_timing + ", CUDA events on the executor stream, best of 3 x 10 replays",
                "gemm_ms_trials": [round(t, 4) for t in trials],
                "gemm_launches_per_step": len(gemm_ops), "gemms_per_step": len(members),
                "gemm_ms_per_step": round(gemm_ms, 4),
                "gemm_share_of_step": round(gemm_ms / ms_per_step, 4),
                "engines": sorted(engines)}
    kern = torch.tensor([ex.kernel_launches() * args.steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(kern)

    cb = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args.cpu_steps, sample_batch=4 if args.workload == "bert" else 2,
                          workload=args.workload)

    if rank == 0:
        samples = batch
        line = {
            "metric": "samples/sec per train iter of HAP program",
            "value": round(samples / (ms_per_step * 1e-3), 2),
            "unit": "samples/s",
            "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": wl["desc"],
                       "global_batch": batch, "seq_len": _seq(args.workload), "parallelism": f"hap-spmd{n}",
                       "plan": plan_name, "sm_caps": caps, "ratios": list(ratios),
                       "grad_sync": dict(sorted(ex.sync_choice.items())) or "n/a (m=1)",
                       "grad_sync_mode": args.grad_sync, "collectives": args.collectives,
                       "collective_impls": ex.collective_impls(),
                       "l2": "inputs larger than L2 (step working set >> 126 MB)",
                       "wgrad_side_stream": dict(zip(("gemm_launches", "forks", "joins"), ex.wgrad_stats)),
                       "tuned_gemm_signatures": getattr(ex, "tuned_signatures", 0)},
            "e2e": {"value": round(samples / (float(e2e_ms.item()) * 1e-3), 2), "unit": "samples/s",
                    "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": 4 * n,
                    "pipeline": "batch i+1 copied H2D (pinned, copy stream) while step i runs; loss "
                                "D2H every step, read on the host one step later"},
            "roofline": roofline,
            "cpu_baseline": None if cb is None else {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "gpu_launches": int(kern.item()),
            "clocks": clk.summary(),
            "loss": losses[0],
        }
        emit_json(line)
    ex.graph = None           # release the captured collectives before the communicator
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ex.close()
    if world > 1:
        dist.destroy_process_group()
    log("done")


if __name__ == "__main__":
    _quiet_stdout()
    main()
