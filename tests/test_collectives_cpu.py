"""The multi-process compile path on CPU: two gloo ranks, each compiling its
rank of every 2-device golden program exactly as a one-process-per-GPU run
does (NcclGroup; gather = NCCL send/recv, NCCL padded or the NVLink kernels;
gradient sync = all-reduce or sufficient-factor broadcasting), then running
the compiled op list on the host (tests/cpu_exec.py: numpy semantics of
every C-ABI entry point, collectives over gloo).  Checks, without a GPU:

* losses and every source gradient against the oracle in fp32 storage
  (parity_common.check: rtol 1e-3) — so per-rank shapes, shard offsets, the
  pack / unpack order of non-leading shard axes and the adjoint collectives
  (all-gather <-> reduce-scatter, all-to-all back) are right;
* both ranks issue the same collective sequence, and every all-to-all's send
  counts match the peer's receive counts (asserted inside the emulation);
* the flat gradient-bucket layout is identical on both ranks, 256-byte
  aligned, non-overlapping and covers every all-reduced gradient.

Reference semantics: interpreter.py:69-101 (collectives), :155-162."""
import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
WORLD = 2
VARIANTS_ALL = [("sendrecv", "all_reduce"), ("kernel", "sfb")]
VARIANTS_SOME = [("padded", "all_reduce"), ("kernel", "all_reduce"), ("sendrecv", "sfb"), ("auto", "auto")]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, out_dir):
    try:
        _work(rank, port, out_dir)
    except BaseException:
        import traceback

        with open(os.path.join(out_dir, f"rank{rank}.err"), "w") as fh:
            fh.write(traceback.format_exc())
        raise


def _work(rank, port, out_dir):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.join(HERE, "multi"))
    import torch.distributed as dist

    import cpu_exec
    import goldens
    from parity_common import cases, check
    from paper_2401_05965_b200.executor import ExecConfig, Executor, NcclGroup
    from paper_2401_05965_b200.program import DistributedProgram
    from paper_2401_05965_b200.sharding import table_from_plan
    from paper_2401_05965_b200 import workloads
    from paper_2401_05965_b200.cost_model import ClusterSpec

    class HostNcclGroup(NcclGroup):
        """Placeholder communicators: the compile path only passes them on."""

        def close(self):
            pass

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    group = HostNcclGroup(rank, WORLD, 1, 2)
    failures, runs = [], 0
    for i, (name, doc, gname, inputs) in enumerate(cases(WORLD)):
        g = goldens.graph(gname)
        shapes = {n.id: n.shape for n in g.sources()}
        refs = {n.id for n in g.sources()}
        for gather, sync in VARIANTS_ALL + (VARIANTS_SOME if i % 4 == 0 else []):
            label = f"{name} {gather} {sync}"
            # "auto": per-call-site NCCL-vs-kernel and SFB-vs-all-reduce choices from the fitted lines on
            # heterogeneous SM caps — every rank must make the same choices
            extra = dict(sm_caps=[148, 104], cluster=ClusterSpec.from_dict(workloads.cluster_doc([148, 104]))) \
                if gather == "auto" else {}
            ex = Executor(DistributedProgram.from_json(doc["program"]), WORLD, table_from_plan(doc), shapes,
                          group=group, config=ExecConfig(dtype="fp32", input_grads=True, gather=gather, grad_sync=sync,
                                                         **extra),
                          device=torch.device("cpu"))
            ex.load(inputs)
            runner = cpu_exec.step(ex)
            runs += 1
            grads = {ref: {r: [(did, t.float().numpy()) for did, t in forms] for r, forms in ex.gradient(ref).items()}
                     for ref in refs}
            failures += check(label, doc, gname, inputs, "fp32", ex.losses(), grads)
            kinds = group.exchange([t[0] for t in runner.trace])
            if any(k != kinds[0] for k in kinds):
                failures.append(f"{label}: ranks issued different collective sequences {kinds}")
            flat = getattr(ex, "_flat", None)
            if flat is not None:
                layout = sorted(flat[1].values())
                if group.exchange(layout)[0] != layout:
                    failures.append(f"{label}: gradient buckets differ across ranks")
                end = -1
                for off, n in layout:
                    if off % 64 or off < end:
                        failures.append(f"{label}: bucket layout misaligned or overlapping at {off}")
                    end = off + n
                synced = {f.output for f in ex._synced_params() if ex._n_contrib.get(f.output, 0) > 0}
                if synced != set(flat[1]):
                    failures.append(f"{label}: buckets {sorted(flat[1])} vs all-reduced {sorted(synced)}")
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as fh:
        fh.write(f"{runs}\n" + "\n".join(failures))
    dist.destroy_process_group()


def test_two_gloo_ranks_compile_and_run_every_two_device_program(tmp_path):
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, str(tmp_path))) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
        if p.is_alive():
            p.kill()
            pytest.fail("gloo worker timed out")
    errs = [(tmp_path / f"rank{r}.err").read_text() for r in range(WORLD) if (tmp_path / f"rank{r}.err").exists()]
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs] + errs
    for r in range(WORLD):
        runs, *failures = (tmp_path / f"rank{r}.txt").read_text().split("\n")
        assert int(runs) > 200, runs
        failures = [f for f in failures if f]
        assert not failures, "\n".join(failures[:30])
