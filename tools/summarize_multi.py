"""Summarise one tools/gpu_multi.sh session (gpurun_out/m<N>/) into a
markdown table for profiles/: fitted collective lines, NVLink byte counters
of the peer-memory kernels, the bench lines of every variant, the parity
result.

    python tools/summarize_multi.py gpurun_out/m2 > profiles/r02_multi_n2.md
"""
import glob
import json
import os
import sys


def _last_json(path):
    try:
        lines = [ln for ln in open(path).read().splitlines() if ln.strip().startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except OSError:
        return None


def main():
    d = sys.argv[1]
    out = []
    status = open(os.path.join(d, "status.txt")).read() if os.path.exists(os.path.join(d, "status.txt")) else ""
    out.append(f"# {os.path.basename(d)} — multi-GPU session (tools/gpu_multi.sh)\n")
    out.append("Exit codes:\n\n```\n" + status.strip() + "\n```\n")
    fit_path = os.path.join(d, "collectives_b200.json")
    if os.path.exists(fit_path):
        fits = json.load(open(fit_path))
        out.append("## Fitted collective lines (cost_model.fit_linear over tools/coll_fit.py sweeps)\n")
        out.append("| world | op | impl | latency us | bandwidth GB/s | residual |")
        out.append("|---|---|---|---:|---:|---:|")
        for world, ops in sorted(fits.items()):
            for op, impls in sorted(ops.items()):
                for impl, v in sorted(impls.items()):
                    out.append(f"| {world} | {op} | {impl} | {v['latency_s'] * 1e6:.2f} | {v['bw_Bps'] / 1e9:.1f} | "
                               f"{v.get('residual_s', 0) * 1e6:.2f} us |")
        out.append("")
    nv = os.path.join(d, "nvl_counters.json")
    if os.path.exists(nv):
        doc = json.load(open(nv))
        out.append("## NVLink data counters around the peer-memory kernels (NVML, per rank)\n")
        out.append(f"SM caps {doc['caps']}; `alg` = bytes the rank must receive / send per call (the larger), "
                   "`counted` = NVLink TX / RX data bytes the GPU's counters moved per call; GB/s over the "
                   "max-over-ranks CUDA-event time of back-to-back calls; frac = alg GB/s / 770 GB/s.\n")
        out.append("| op | rows | rank | us/call | alg rx MB | alg tx MB | counted tx MB | counted rx MB | alg GB/s | "
                   "counted GB/s | frac of 770 |")
        out.append("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
        for r in doc["ranks"]:
            if "us_per_call_max_over_ranks" not in r:
                continue
            out.append(f"| {r['op']} | {r['rows']} | {r['rank']} | {r['us_per_call_max_over_ranks']} | "
                       f"{r['rx_bytes'] / 1e6:.1f} | {r['tx_bytes'] / 1e6:.1f} | {r['nvlink_tx_bytes_counted'] / 1e6:.1f} | "
                       f"{r['nvlink_rx_bytes_counted'] / 1e6:.1f} | {r['alg_GBps']} | {r['counted_GBps']} | "
                       f"{r['frac_of_770']} |")
        out.append("")
    out.append("## Bench lines (bench.py under torchrun)\n")
    out.append("| variant | samples/s | ms/step | e2e samples/s | roofline bound | frac | grad sync | collectives |")
    out.append("|---|---:|---:|---:|---|---:|---|---|")
    for path in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
        line = _last_json(path)
        tag = os.path.basename(path)[6:-5]
        if not line:
            out.append(f"| {tag} | (no line) | | | | | | |")
            continue
        rf = line.get("roofline") or {}
        cfg = line.get("config") or {}
        ex = line.get("executor") or {}
        out.append(f"| {tag} | {line['value']:.1f} | {line['ms_per_step']:.3f} | {line['e2e']['value']:.1f} | "
                   f"{rf.get('bound')} | {rf.get('frac')} | {cfg.get('grad_sync_mode')} | "
                   f"{cfg.get('collectives', ex.get('collectives'))} |")
    out.append("")
    par = os.path.join(d, "parity.log")
    if os.path.exists(par):
        tail = [ln for ln in open(par).read().splitlines() if "parity" in ln.lower() or "FAIL" in ln][-6:]
        out.append("## NCCL-group parity (tests/multi/nccl_parity.py)\n\n```\n" + "\n".join(tail) + "\n```\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
