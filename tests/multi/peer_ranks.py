"""The multi-device path on ONE GPU: every golden program for 2 and 3
devices (the reference planner's plans and the enumerated programs with
collectives) executed by m program ranks inside one process — each rank an
Executor on its own stream, SM cap 148 // m, built and stepped in its own
thread — whose collectives are only the hand-written NVLink peer-memory
kernels (PeerGroup, in-process form): push all-gather, direct reduce-scatter,
two-shot all-reduce, push all-to-all, the SFB factor gathers on the side
stream and the bucketed gradient all-reduce.  Checked against the CPU oracle
(parity_common.check), and in fp32 against the single-executor LocalGroup run
of the same program bit for bit (the peer kernels sum in rank order, as the
LocalGroup does).  Run by tests/test_gpu_peer_ranks.py in a subprocess with a
timeout:

    python tests/multi/peer_ranks.py [substring] [--world 2,3] [--variants all_reduce,sfb]
"""
import argparse
import os
import sys
import time

# every rank's streams on their own hardware work queues (see
# paper_2401_05965_b200/__init__.py); before CUDA is initialised
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import goldens  # noqa: E402
from oracle import interpreter_np as O  # noqa: E402
from parity_common import cases, check  # noqa: E402
from paper_2401_05965_b200.executor import (ExecConfig, Executor, LocalGroup, run_ranks,  # noqa: E402
                                            thread_peer_groups)
from paper_2401_05965_b200.program import DistributedProgram  # noqa: E402
from paper_2401_05965_b200.sharding import table_from_plan  # noqa: E402


def grads_of(exs, program):
    refs = {ins.ref for ins in program.instrs if ins.kind.startswith(("parameter", "placeholder"))}
    out = {}
    for ref in refs:
        per = {}
        for ex in exs:
            for r, forms in ex.gradient(ref).items():
                per[r] = [(did, t.float().cpu().numpy()) for did, t in forms]
        out[ref] = per
    return out


def run_peer(doc, shapes, inputs, dtype, sync, capture):
    prog = DistributedProgram.from_json(doc["program"])
    m = int(doc["devices"])
    table = table_from_plan(doc)
    caps = [148 // m] * m
    groups = thread_peer_groups(m)
    exs = run_ranks([lambda r=r: Executor(prog, m, table, shapes, group=groups[r],
                                          config=ExecConfig(dtype=dtype, sm_caps=caps, input_grads=True,
                                                            grad_sync=sync))
                     for r in range(m)])
    LIVE[:] = exs
    run_ranks([lambda ex=ex: ex.load(inputs) for ex in exs])
    if capture:
        run_ranks([lambda ex=ex: ex.step() for ex in exs])   # warm up together, capture one by one
        for ex in exs:
            ex.capture(warmup=False)
        run_ranks([lambda ex=ex: ex.load(inputs) for ex in exs])
    run_ranks([lambda ex=ex: ex.step() for ex in exs])
    torch.cuda.synchronize()
    losses = run_ranks([lambda ex=ex: ex.losses() for ex in exs])[0]
    return exs, losses


def run_local(doc, shapes, inputs, dtype, sync):
    m = int(doc["devices"])
    ex = Executor(DistributedProgram.from_json(doc["program"]), m, table_from_plan(doc), shapes, group=LocalGroup(m),
                  config=ExecConfig(dtype=dtype, sm_caps=[148 // m] * m, input_grads=True, grad_sync=sync))
    ex.load(inputs)
    ex.step()
    torch.cuda.synchronize()
    return ex, ex.losses()


LIVE: list = []   # executors of the current run (the watchdog's view)


def _dump_signal_pages():
    """Each rank's peer-memory signal pages (p2p.cu SignalPage: ready, done,
    armed per peer, epoch, grid-barrier counters), read through a private
    non-blocking stream while the kernels spin (hap_symm_peek)."""
    import ctypes

    import numpy as np

    from paper_2401_05965_b200 import _lib

    L = _lib.lib()
    m = len(LIVE)
    for r, ex in enumerate(LIVE):
        for tag, ctx in ex.__dict__.get("_symm", {}).items():
            buf = (ctypes.c_uint64 * 64)()
            st = L.hap_symm_peek(ctx, buf)
            a = np.frombuffer(buf, dtype=np.uint64)
            gen = (int(a[49]) >> 32, int(a[49]) & 0xffffffff)
            print(f"[watchdog] rank {r} {tag} page (status {st}): ready {a[0:m].tolist()} done {a[16:16 + m].tolist()} "
                  f"armed {a[32:32 + m].tolist()} epoch {int(a[48])} barrier (generation, arrive) {gen}", flush=True)


def _install_watchdog(args):
    """--verbose: every eager op is followed by a CUDA event; when no rank
    makes progress for 30 s, print each rank's first incomplete op, the GPU
    utilisation (a spinning kernel or a host-side wait), and exit 3."""
    import subprocess
    import threading

    from paper_2401_05965_b200 import _lib

    args.capture_every = 0   # events cannot be recorded inside a graph capture

    def run_traced(self, ops):
        trace = self.__dict__.setdefault("op_trace", [])
        for op in ops:
            st = op.fn(*op.args)
            if st:
                _lib.check(st, op.what)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            trace.append((op.what, ev))

    Executor._run = run_traced

    def watch():
        last, since = None, time.time()
        while True:
            threading.Event().wait(5)
            state = []
            for r, ex in enumerate(list(LIVE)):
                trace = list(ex.__dict__.get("op_trace", []))
                first = next((i for i, (_, ev) in enumerate(trace) if not ev.query()), None)
                state.append((r, len(trace), first, trace[first][0] if first is not None else "-"))
            if state != last:
                last, since = state, time.time()
                continue
            if time.time() - since < 30 or not state or all(f is None for _, _, f, _ in state):
                continue
            util = subprocess.run(["nvidia-smi", "--query-gpu=utilization.gpu", "--format=csv,noheader"],
                                  capture_output=True, text=True).stdout.strip()
            for r, n, first, what in state:
                print(f"[watchdog] rank {r}: {n} ops enqueued, first incomplete op #{first}: {what}", flush=True)
                trace = LIVE[r].__dict__.get("op_trace", [])
                lo = max(0, (first or 0) - 4)
                print(f"[watchdog]   ops {lo}..: {[w for w, _ in trace[lo:(first or 0) + 3]]}", flush=True)
            # the page dump goes through the CUDA runtime, which a stalled
            # GPU can block: bounded, then exit regardless
            dumper = threading.Thread(target=_dump_signal_pages, daemon=True)
            dumper.start()
            dumper.join(10)
            print(f"[watchdog] GPU utilisation {util}; exiting", flush=True)
            os._exit(3)

    threading.Thread(target=watch, daemon=True).start()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("only", nargs="?")
    ap.add_argument("--world", default="2,3")
    ap.add_argument("--variants", default="all_reduce,sfb")
    ap.add_argument("--dtypes", default="fp32,bf16")
    ap.add_argument("--capture-every", type=int, default=5, help="every k-th run replays a captured graph (0: never)")
    ap.add_argument("--stride", type=int, default=1, help="every k-th case only")
    ap.add_argument("--rotate", action="store_true",
                    help="one (dtype, gradient sync) combination per case, rotating through them")
    ap.add_argument("--skip", default="", help="comma-separated dtype:sync combinations to leave out")
    ap.add_argument("--start-run", type=int, default=1, help="skip the runs before this one (resume)")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    if args.verbose:
        _install_watchdog(args)
    torch.cuda.set_device(0)
    failures, count, bit_equal, bit_total = [], 0, 0, 0
    skip = {tuple(c.split(":")) for c in args.skip.split(",") if c}
    combos = [(d, v) for d in args.dtypes.split(",") for v in args.variants.split(",") if (d, v) not in skip]
    t0 = time.time()
    for world in [int(w) for w in args.world.split(",")]:
        for ci, (name, doc, gname, inputs) in enumerate(cases(world)):
            if args.only and args.only not in name:
                continue
            if ci % args.stride:
                continue
            g = goldens.graph(gname)
            shapes = {n.id: n.shape for n in g.sources()}
            program, _, _ = O.load_plan(doc)
            for dtype, sync in ([combos[(ci // args.stride) % len(combos)]] if args.rotate else combos):
                count += 1
                if count < args.start_run:
                    continue
                label = f"{name} {dtype} {sync}"
                capture = args.capture_every > 0 and count % args.capture_every == 0
                if args.verbose:
                    print(f"run {count} [{time.time() - t0:.1f}s]: {label}{' (graph)' if capture else ''}", flush=True)
                try:
                    exs, losses = run_peer(doc, shapes, inputs, dtype, sync, capture)
                except Exception as exc:  # noqa: BLE001 - fatal: a peer kernel may be left spinning
                    # one rank failed to enqueue its step: the other rank's peer kernel now waits for a
                    # partner that never comes, so no later GPU call can return — report and stop
                    import traceback

                    print(f"  FAIL {label}: {type(exc).__name__}: {exc}\n{traceback.format_exc()}", flush=True)
                    for f in failures[:40]:
                        print("  FAIL", f, flush=True)
                    os._exit(2)
                grads = grads_of(exs, program)
                failures += check(label + (" graph" if capture else ""), doc, gname, inputs, dtype, losses, grads)
                if dtype == "fp32":
                    lex, llosses = run_local(doc, shapes, inputs, dtype, sync)
                    lgrads = grads_of([lex], program)
                    same = list(losses) == list(llosses) and all(
                        all(np.array_equal(a[1], b[1]) for a, b in zip(grads[ref][r], lgrads[ref][r]))
                        for ref in grads for r in grads[ref])
                    bit_total += 1
                    bit_equal += int(same)
                    lex.close()
                for ex in exs:
                    ex.close()
                print(f"DONE {count}", flush=True)
    print(f"peer ranks parity: {count} runs, {len(failures)} failures; fp32 bit-identical to LocalGroup "
          f"in {bit_equal}/{bit_total}; {time.time() - t0:.0f} s")
    for f in failures[:40]:
        print("  FAIL", f)
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
