"""Where one SM-pair GEMM launch spends its time: per-CTA %globaltimer
stamps from the HAP_GEMM_TRACE build (python -m paper_2401_05965_b200.build
--variant trace), relative to the earliest CTA entry, min / median / max over
the CTAs, next to the launch's CUDA-event time.

    python tools/gemm_trace.py [--json PATH]
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("HAP_LIB_PATH", os.path.join(ROOT, "paper_2401_05965_b200", "libhap_b200_trace.so"))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2401_05965_b200 import _lib  # noqa: E402
from paper_2401_05965_b200._lib import BF16, F32, check  # noqa: E402

EVENTS = {0: "entry", 1: "prologue done", 29: "producer starts", 27: "first K block (cursor done)",
          28: "first stage armed", 2: "first TMA issued", 3: "first MMA (stage full)",
          10: "last unit's first MMA", 9: "last TMA issued", 4: "last MMA commit", 5: "first tile in epilogue",
          11: "last tile in epilogue", 6: "last stores issued", 7: "stores complete", 8: "exit"}
EPI_STEPS = {20: "plain boxes", 16: "plain wait staging read", 17: "plain tcgen05.ld",
             18: "plain convert+st.shared", 19: "plain TMA issue", 26: "fused chunks",
             21: "fused input-load wait", 22: "fused wait staging read", 23: "fused tcgen05.ld",
             24: "fused compute+st.shared", 25: "fused TMA issue"}
WAITS = {12: "MMA waits for data", 13: "MMA waits for TMEM", 14: "TMA waits for a free stage",
         15: "epilogue waits for a tile"}


def main():
    L = _lib.lib()
    L.hap_gemm_trace_set.argtypes = [ctypes.c_void_p, ctypes.c_int]
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream()
    buf = torch.zeros(148 * 32, dtype=torch.int64, device=dev)
    shapes = [("one tile 256x192x64", 256, 192, 64, 0, 0, "none"),
              ("one tile 256x192x768", 256, 192, 768, 0, 0, "none"),
              ("8192x768x768 NN", 8192, 768, 768, 0, 0, "none"), ("8192x768x768 NN add2", 8192, 768, 768, 0, 0, "add2"),
              ("8192x768x3072 NN", 8192, 768, 3072, 0, 0, "none"),
              ("8192x768x3072 NN add2", 8192, 768, 3072, 0, 0, "add2"),
              ("8192x768x3072 NT add", 8192, 768, 3072, 0, 1, "add"),
              ("8192x3072x768 NN", 8192, 3072, 768, 0, 0, "none"),
              ("8192x3072x768 NN swish", 8192, 3072, 768, 0, 0, "swish"),
              ("8192x3072x768 NT swish_bwd", 8192, 3072, 768, 0, 1, "swish_bwd"),
              ("dW 768x3072x8192 TN f32", 768, 3072, 8192, 1, 0, "none")]
    EPI = {"none": _lib.EPI_NONE, "add": _lib.EPI_ADD, "add2": _lib.EPI_ADD2, "swish": _lib.EPI_SWISH,
           "swish_bwd": _lib.EPI_SWISH_BWD}
    _lib.load_tune_table()
    out = []
    for name, M, N, K, ta, tb, epi in shapes:
        a = torch.randn((K, M) if ta else (M, K), device=dev).to(torch.bfloat16)
        b = torch.randn((N, K) if tb else (K, N), device=dev).to(torch.bfloat16)
        c = torch.empty((M, N), device=dev, dtype=torch.float32 if ta else torch.bfloat16)
        t1, t2, t3 = (torch.randn(M, N, device=dev).to(torch.bfloat16) for _ in range(3))
        d = _lib.GemmDesc()
        d.A, d.lda, d.transA, d.B, d.ldb, d.transB = a.data_ptr(), a.shape[1], ta, b.data_ptr(), b.shape[1], tb
        d.C, d.ldc, d.M, d.N, d.K = c.data_ptr(), N, M, N, K
        e = EPI[epi]
        d.epi, d.epi_tag = e, _lib.UNARY_TAGS["sigmoid"]
        if e in (_lib.EPI_ADD, _lib.EPI_ADD2, _lib.EPI_SWISH_BWD):
            d.R, d.ldr = t1.data_ptr(), N
        if e == _lib.EPI_SWISH_BWD:
            d.R2, d.ldr2 = t2.data_ptr(), N
        if e in (_lib.EPI_ADD2, _lib.EPI_SWISH):
            d.Y, d.ldy = t2.data_ptr(), N
        if e == _lib.EPI_SWISH:
            d.Z, d.ldz = t3.data_ptr(), N
        arr = (_lib.GemmDesc * 1)(d)
        odt = F32 if ta else BF16

        def run():
            check(L.hap_matmul_batch(arr, 1, 0, BF16, odt, 0, s.cuda_stream))

        L.hap_gemm_trace_set(None, 0)
        with torch.cuda.stream(s):
            for _ in range(5):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                run()
            e1.record(s)
        torch.cuda.synchronize()
        ev_us = e0.elapsed_time(e1) * 1e3 / 20
        runs = []
        for _ in range(5):
            buf.zero_()
            torch.cuda.synchronize()
            L.hap_gemm_trace_set(ctypes.c_void_p(buf.data_ptr()), 148)
            with torch.cuda.stream(s):
                run()
            torch.cuda.synchronize()
            L.hap_gemm_trace_set(None, 0)
            t = buf.view(148, 32).cpu()
            runs.append(t)
        t = runs[-1]
        ctas = int((t[:, 0] > 0).sum())
        if ctas == 0:
            print(f"\n{name}: not the SM-pair kernel (no trace), {ev_us:.2f} us per launch")
            out.append({"name": name, "event_us": round(ev_us, 2), "ctas": 0})
            continue
        t0 = int(t[:ctas, 0].min())
        row = {"name": name, "event_us": round(ev_us, 2), "ctas": ctas, "events": {}}
        print(f"\n{name}: {ctas} CTAs, back-to-back event time {ev_us:.2f} us per launch")
        for ev, label in EVENTS.items():
            col = t[:ctas, ev]
            col = col[col > 0]
            if len(col) == 0:
                continue
            rel = (col - t0).double() / 1e3
            q = (round(float(rel.min()), 2), round(float(rel.median()), 2), round(float(rel.max()), 2))
            row["events"][label] = q
            print(f"  {label:26s} min {q[0]:8.2f}  med {q[1]:8.2f}  max {q[2]:8.2f} us  (n={len(col)})")
        for ev, label in WAITS.items():
            col = t[:ctas, ev]
            if ev in (12, 13):
                col = col[0::2]   # leader CTAs issue the MMAs
            w = col.double() / 1e3
            q = (round(float(w.min()), 2), round(float(w.median()), 2), round(float(w.max()), 2))
            row["events"][label] = q
            print(f"  {label:26s} min {q[0]:8.2f}  med {q[1]:8.2f}  max {q[2]:8.2f} us total per CTA")
        for ev, label in EPI_STEPS.items():
            col = t[:ctas, ev].double()
            if float(col.max()) <= 0:
                continue
            w = col if ev in (20, 26) else col / 1e3
            q = (round(float(w.min()), 2), round(float(w.median()), 2), round(float(w.max()), 2))
            row["events"][label] = q
            print(f"  {label:26s} min {q[0]:8.2f}  med {q[1]:8.2f}  max {q[2]:8.2f} {'' if ev in (20, 26) else 'us'}"
                  " (one epilogue warp)")
        out.append(row)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
