"""Multi-process parity: every m=2 golden program (plans and enumerated
programs with collectives) executed with one process per GPU over NCCL,
checked against the CPU oracle.  Launched by tests/test_gpu_multi.py as

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/multi/nccl_parity.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import goldens  # noqa: E402
from oracle import interpreter_np as O  # noqa: E402
from parity_common import cases, check  # noqa: E402
from paper_2401_05965_b200.executor import ExecConfig, Executor, NcclGroup  # noqa: E402
from paper_2401_05965_b200.program import DistributedProgram  # noqa: E402
from paper_2401_05965_b200.sharding import table_from_plan  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    group = NcclGroup.from_torch_distributed()
    failures, count = [], 0
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for name, doc, gname, inputs in cases(world):
        if only and only not in name:
            continue
        g = goldens.graph(gname)
        shapes = {n.id: n.shape for n in g.sources()}
        program, m, table = O.load_plan(doc)
        # Gradient sync: all-reduce for every gather implementation, plus
        # sufficient-factor broadcasting through the P2P and send/recv gathers.
        variants = [(g_, "all_reduce") for g_ in ("kernel", "padded", "sendrecv")]
        variants += [("kernel", "sfb"), ("sendrecv", "sfb"), ("auto", "all_reduce")]
        if os.environ.get("HAP_PARITY_VARIANTS"):
            variants = [tuple(v.split(":")) for v in os.environ["HAP_PARITY_VARIANTS"].split(",")]
        overlap = os.environ.get("HAP_PARITY_OVERLAP", "1") == "1"
        for dtype in ("fp32", "bf16"):
            for gather, sync in variants:
                count += 1
                ex = Executor(DistributedProgram.from_json(doc["program"]), m, table_from_plan(doc), shapes,
                              group=group, config=ExecConfig(dtype=dtype, input_grads=True, gather=gather,
                                                             grad_sync=sync, overlap_sfb=overlap))
                ex.load(inputs)
                ex.step()
                torch.cuda.synchronize()
                losses = ex.losses()
                grads = {ref: {r: [(did, t.float().cpu().numpy()) for did, t in forms]
                               for r, forms in ex.gradient(ref).items()}
                         for ref in {ins.ref for ins in program.instrs if ins.kind.startswith(("parameter", "placeholder"))}}
                failures += check(f"{name} {dtype} {gather} {sync}", doc, gname, inputs, dtype, losses, grads)
                ex.group = None  # the communicator is shared across executors
    fl = [None] * world
    dist.all_gather_object(fl, failures)
    if rank == 0:
        allf = [f for sub in fl for f in sub]
        print(f"nccl parity: {count} runs per rank, {len(allf)} failures")
        for f in allf[:40]:
            print("  FAIL", f)
    group.close()
    dist.destroy_process_group()
    sys.exit(1 if any(fl) else 0)


if __name__ == "__main__":
    main()
