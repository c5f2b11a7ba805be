"""Where a multi-GPU training step spends its time (run with torchrun like
bench.py): the captured step, then the forward, the backward+update with
and without the gradient collectives, and the collectives alone — each
replayed as its own CUDA graph, max over ranks.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/step_breakdown.py [--workload bert|moe]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2401_05965_b200 import workloads  # noqa: E402
from paper_2401_05965_b200.cost_model import ClusterSpec  # noqa: E402
from paper_2401_05965_b200.executor import ExecConfig, Executor, NcclGroup  # noqa: E402
from paper_2401_05965_b200.program import DistributedProgram  # noqa: E402
from paper_2401_05965_b200.sharding import table_from_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bert")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    wl = bench.WORKLOADS[args.workload]
    caps = workloads.sm_caps(world)
    g = bench._graph(args.workload, wl["per_gpu_batch"] * world)
    doc = bench._plan_doc(args.workload, world)
    ex = Executor(DistributedProgram.from_json(doc["program"]), world, table_from_plan(doc),
                  {n.id: n.shape for n in g.sources()}, group=NcclGroup.from_torch_distributed(),
                  config=ExecConfig(dtype="bf16", sm_caps=caps, lr=bench.LR,
                                    cluster=ClusterSpec.from_dict(workloads.cluster_doc(caps)),
                                    ratios=tuple(doc["ratios"][0])), device=dev)
    ex.load(workloads.synthetic_inputs(g, 0, scaled=True))
    ex.step()
    torch.cuda.synchronize(dev)
    comm_names = ("hap_all_reduce", "hap_all_gather_v", "hap_p2p_all_gather_v", "hap_reduce_scatter_v",
                  "hap_p2p_reduce_scatter_v", "hap_all_to_all_v", "hap_grouped_broadcast")

    def timed(ops_list, label):
        graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize(dev)
        dist.barrier()
        with torch.cuda.graph(graph, stream=ex.stream, capture_error_mode="thread_local"):
            for ops in ops_list:
                ex._run(ops)
        torch.cuda.synchronize(dev)
        dist.barrier()
        with torch.cuda.stream(ex.stream):
            graph.replay()
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ex.stream)
        with torch.cuda.stream(ex.stream):
            for _ in range(args.reps):
                graph.replay()
        e1.record(ex.stream)
        torch.cuda.synchronize(dev)
        t = torch.tensor([e0.elapsed_time(e1) / args.reps], device=dev)
        ts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(ts, t)
        if rank == 0:
            print(f"{label:44s} " + " ".join(f"{float(x):7.3f}" for x in ts) + " ms (per rank)", flush=True)
        del graph

    is_comm = lambda op: op.what in comm_names  # noqa: E731
    bwd_nocomm = [op for op in ex.ops_bwd if not is_comm(op)]
    comm_only = [op for op in ex.ops_fwd + ex.ops_bwd if is_comm(op) or op.what in ("event.record", "stream.wait_event")]
    timed([ex.ops_fwd, ex.ops_bwd, ex.ops_upd], "step (fwd+bwd+sync+update)")
    timed([ex.ops_fwd], "forward")
    timed([ex.ops_bwd, ex.ops_upd], "backward + sync + update")
    timed([bwd_nocomm, ex.ops_upd], "backward + update, collectives removed")
    timed([comm_only], "collectives alone (same streams)")
    if rank == 0:
        n_comm = sum(1 for op in ex.ops_fwd + ex.ops_bwd if is_comm(op))
        print(f"collective launches per step: {n_comm}; grad sync: {sorted(set(ex.sync_choice.values()))}")
    torch.cuda.synchronize(dev)
    dist.barrier()
    ex.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
