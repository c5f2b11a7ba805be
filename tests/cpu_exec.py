"""Host emulation of a compiled executor op list — TEST INFRASTRUCTURE.

The executor compiles a program into a flat list of C-ABI launches
(executor.Op) with every pointer and size resolved.  On a host without a GPU
the executor can still COMPILE (device "cpu": buffers in host memory, streams
and events are stubs — executor._HostStream).  This module then runs that op
list with numpy, one op at a time, giving each C-ABI entry point the
semantics include/hap_b200.h documents, and the collectives through
torch.distributed (gloo).  tests/test_collectives_cpu.py uses it with two
gloo ranks to check the multi-process compile path — per-rank shapes,
collective counts and offsets, pack / unpack order of non-leading shard axes,
the adjoint collectives, SFB factor gathers and the gradient-bucket layout —
against the oracle, without a GPU.  fp32 programs only (numpy has no bf16).
"""
from __future__ import annotations

import ctypes
import math
import struct

import numpy as np
import torch
import torch.distributed as dist

from paper_2401_05965_b200 import _lib

_UNARY = {0: np.exp, 1: np.negative, 2: lambda x: np.maximum(x, 0.0),
          3: lambda x: 1.0 / (1.0 + np.exp(-x)), 4: np.tanh}


def _deriv(tag, x, y):
    if tag == 0:
        return y
    if tag == 1:
        return -np.ones_like(x)
    if tag == 2:
        return (x > 0).astype(np.float64)
    if tag == 3:
        return y * (1.0 - y)
    return 1.0 - y * y


class Memory:
    """Pointer -> float32 numpy view over every host tensor the executor owns."""

    def __init__(self, ex):
        self.spans = []
        seen = set()
        tensors = [b.tensor for b in ex._pool] + [t for t in ex.__dict__.get("_keepalive", [])
                                                   if isinstance(t, torch.Tensor)]
        for t in tensors:
            st = t.untyped_storage()
            base = st.data_ptr()
            if base in seen or st.nbytes() == 0:
                continue
            seen.add(base)
            self.spans.append((base, base + st.nbytes()))
        self.spans.sort()

    def view(self, ptr: int, n: int) -> np.ndarray:
        if n == 0:
            return np.zeros(0, dtype=np.float32)
        for lo, hi in self.spans:
            if lo <= ptr and ptr + 4 * n <= hi:
                return np.ctypeslib.as_array((ctypes.c_float * max(n, 1)).from_address(ptr))[:n]
        raise KeyError(f"pointer {ptr:#x} (+{n} floats) is not inside an executor buffer")

    def mat(self, ptr: int, rows: int, cols: int, ld: int) -> np.ndarray:
        if rows == 0 or cols == 0:
            return np.zeros((rows, cols), dtype=np.float32)
        flat = self.view(ptr, (rows - 1) * ld + cols)
        return np.lib.stride_tricks.as_strided(flat, shape=(rows, cols), strides=(ld * 4, 4))


def _arr(a, n=None):
    """ctypes int64 array argument -> list."""
    return [int(v) for v in (a if n is None else a[:n])]


def _store(dst: np.ndarray, value, accumulate: int):
    if accumulate:
        dst[...] = dst + value
    else:
        dst[...] = value


class HostRunner:
    """Runs an executor's op list on the host; collectives over the default
    torch.distributed group (one process per program rank)."""

    def __init__(self, ex):
        if ex.wdt != _lib.F32:
            raise ValueError("host emulation runs fp32 programs only")
        self.ex = ex
        self.mem = Memory(ex)
        self.rank = ex.group.rank
        self.m = ex.m
        self.trace = []           # (op name, per-call detail) of every collective, in order

    # ---- collectives over gloo (object exchange: small test tensors)
    def _gather(self, obj):
        return self.ex.group.exchange(obj)

    def run(self, ops):
        for op in ops:
            name = op.what
            if name in ("event.record", "stream.wait_event"):
                continue
            fn = getattr(self, "hap_matmul_batch" if op.gemm is not None else name, None)
            if fn is None:
                raise NotImplementedError(f"no host semantics for {name}")
            if op.meta is not None:
                fn(**op.meta)
            else:
                fn(*op.args)

    # ---- compute
    def hap_matmul_batch(self, descs, count, sum_k, in_dt, out_dt, cap, stream):
        m = self.mem
        total = None
        for q in range(count):
            d = descs[q]
            if d.epi:
                raise NotImplementedError("fused epilogues are bf16-only")
            a = m.mat(d.A, d.K, d.M, d.lda).T if d.transA else m.mat(d.A, d.M, d.K, d.lda)
            b = m.mat(d.B, d.N, d.K, d.ldb).T if d.transB else m.mat(d.B, d.K, d.N, d.ldb)
            prod = a.astype(np.float64) @ b.astype(np.float64)
            if sum_k:
                total = prod if total is None else total + prod
            else:
                _store(m.mat(d.C, d.M, d.N, d.ldc), prod, d.accumulate)
        if sum_k:
            d = descs[0]
            _store(m.mat(d.C, d.M, d.N, d.ldc), total, d.accumulate)

    def hap_unary(self, tag, x, xdt, y, ydt, n, cap, stream):
        self.mem.view(y, n)[...] = _UNARY[tag](self.mem.view(x, n).astype(np.float64))

    def hap_unary_grad(self, tag, x, y, xydt, dy, dydt, dx, dxdt, n, acc, cap, stream):
        v = self.mem.view
        xv, yv = v(x, n).astype(np.float64), v(y, n).astype(np.float64)
        _store(v(dx, n), v(dy, n) * _deriv(tag, xv, yv), acc)

    def hap_binary(self, tag, a, b, in_dt, out, out_dt, n, cap, stream):
        v = self.mem.view
        av, bv = v(a, n).astype(np.float64), v(b, n).astype(np.float64)
        v(out, n)[...] = av + bv if tag == 0 else av * bv

    def hap_mul_grad(self, a, b, in_dt, dy, dydt, da, db, d_dt, n, acc, cap, stream):
        v = self.mem.view
        av, bv, g = v(a, n).astype(np.float64), v(b, n).astype(np.float64), v(dy, n).astype(np.float64)
        if da and db and da == db:
            _store(v(da, n), g * bv + g * av, acc)
            return
        if da:
            _store(v(da, n), g * bv, acc)
        if db:
            _store(v(db, n), g * av, acc)

    def hap_swish_fwd(self, tag, x, y, z, dt, n, cap, stream):
        v = self.mem.view
        xv = v(x, n).astype(np.float64)
        yv = _UNARY[tag](xv)
        v(y, n)[...] = yv
        v(z, n)[...] = xv * v(y, n)

    def hap_swish_bwd(self, tag, x, y, dz, dx, dt, n, acc, cap, stream):
        v = self.mem.view
        xv, yv, g = v(x, n).astype(np.float64), v(y, n).astype(np.float64), v(dz, n).astype(np.float64)
        _store(v(dx, n), g * yv + (g * xv) * _deriv(tag, xv, yv), acc)

    def hap_gate_fwd(self, tag, a, b, c, p, q, o, dt, n, cap, stream):
        v = self.mem.view
        v(p, n)[...] = v(a, n).astype(np.float64) * v(b, n)
        v(q, n)[...] = _UNARY[tag](v(p, n).astype(np.float64))
        v(o, n)[...] = v(q, n).astype(np.float64) * v(c, n)

    def hap_gate_bwd(self, tag, a, b, c, p, q, dout, da, db, dc, dt, n, acc_a, acc_b, acc_c, cap, stream):
        v = self.mem.view
        av, bv, cv = (v(t, n).astype(np.float64) for t in (a, b, c))
        pv, qv, g = v(p, n).astype(np.float64), v(q, n).astype(np.float64), v(dout, n).astype(np.float64)
        if dc:
            _store(v(dc, n), g * qv, acc_c)
        dp = (g * cv) * _deriv(tag, pv, qv)
        if da:
            _store(v(da, n), dp * bv, acc_a)
        if db:
            _store(v(db, n), dp * av, acc_b)

    def hap_reduce(self, x, xdt, shape, rank, mask, y, ydt, acc, cap, stream):
        dims = _arr(shape, rank) if rank else []
        xv = self.mem.view(x, math.prod(dims)).reshape(dims).astype(np.float64)
        axes = tuple(d for d in range(rank) if mask >> d & 1)
        out = xv.sum(axis=axes) if axes else xv
        _store(self.mem.view(y, int(np.size(out))).reshape(np.shape(out)), out, acc)

    def hap_unreduce(self, dy, dydt, shape, rank, mask, dx, dxdt, acc, cap, stream):
        dims = _arr(shape, rank) if rank else []
        kept = [e for d, e in enumerate(dims) if not (mask >> d & 1)]
        g = self.mem.view(dy, math.prod(kept)).reshape(kept).astype(np.float64)
        for d in range(rank):
            if mask >> d & 1:
                g = np.expand_dims(g, d)
        _store(self.mem.view(dx, math.prod(dims)).reshape(dims), np.broadcast_to(g, dims), acc)

    def hap_copy_block(self, src, sdt, se, soff, dst, ddt, de, doff, outer, count, inner, acc, cap, stream):
        if outer * count * inner == 0:
            return
        s = self.mem.view(src, outer * se * inner).reshape(outer, se, inner)
        d = self.mem.view(dst, outer * de * inner).reshape(outer, de, inner)
        _store(d[:, doff:doff + count, :], s[:, soff:soff + count, :], acc)

    def hap_axpy(self, alpha, x, xdt, y, ydt, n, acc, cap, stream):
        _store(self.mem.view(y, n), alpha * self.mem.view(x, n).astype(np.float64), acc)

    def hap_fill(self, y, ydt, value, n, stream):
        self.mem.view(y, n)[...] = value

    def hap_sgd_multi(self, table, count, chunks, wdt, lr, cap, stream):
        raw = ctypes.string_at(table, 40 * count)
        for i in range(count):
            mst, grad, w, n, _ = struct.unpack_from("<QQQqq", raw, 40 * i)
            mv = self.mem.view(mst, n)
            mv[...] = mv - np.float32(lr) * self.mem.view(grad, n)
            self.mem.view(w, n)[...] = mv

    # ---- NCCL entry points
    def hap_all_reduce(self, comm, send, recv, count, dt, stream):
        parts = self._gather(np.array(self.mem.view(send, count), dtype=np.float64))
        self.trace.append(("all_reduce", count))
        self.mem.view(recv, count)[...] = sum(parts[1:], parts[0])

    def hap_all_gather_v(self, comm, send, recv, counts, dt, padded, scratch, stream):
        cnt = _arr(counts, self.m)
        parts = self._gather(np.array(self.mem.view(send, cnt[self.rank]), dtype=np.float32))
        self.trace.append(("all_gather_v", tuple(cnt)))
        assert [len(p) for p in parts] == cnt, (cnt, [len(p) for p in parts])
        self.mem.view(recv, sum(cnt))[...] = np.concatenate(parts) if parts else []

    def hap_grouped_broadcast(self, comm, send, recv, counts, dt, stream):
        self.hap_all_gather_v(comm, send, recv, counts, dt, 0, None, stream)

    def hap_reduce_scatter_v(self, comm, send, recv, counts, dt, scratch, stream):
        cnt = _arr(counts, self.m)
        parts = self._gather(np.array(self.mem.view(send, sum(cnt)), dtype=np.float64))
        self.trace.append(("reduce_scatter_v", tuple(cnt)))
        off = sum(cnt[:self.rank])
        total = sum(parts[1:], parts[0])
        self.mem.view(recv, cnt[self.rank])[...] = total[off:off + cnt[self.rank]]

    def hap_all_to_all_v(self, comm, send, scounts, recv, rcounts, dt, stream):
        sc, rc = _arr(scounts, self.m), _arr(rcounts, self.m)
        flat = np.array(self.mem.view(send, sum(sc)), dtype=np.float32)
        chunks = np.split(flat, np.cumsum(sc)[:-1])
        everyone = self._gather([c for c in chunks])
        self.trace.append(("all_to_all_v", tuple(sc), tuple(rc)))
        mine = [everyone[j][self.rank] for j in range(self.m)]
        assert [len(c) for c in mine] == rc, (rc, [len(c) for c in mine])
        self.mem.view(recv, sum(rc))[...] = np.concatenate(mine)

    # ---- NVLink peer-memory kernels (executor Op.meta)
    def _block_of(self, buf, outer, rows, inner):
        return self.mem.view(buf.ptr, outer * rows * inner).reshape(outer, rows, inner)

    def hap_p2p_all_gather_push(self, send, recv, outer, inner, extent, sizes):
        offs = np.cumsum([0] + sizes)
        parts = self._gather(np.array(self._block_of(send, outer, sizes[self.rank], inner)))
        self.trace.append(("p2p_all_gather", tuple(sizes)))
        out = self._block_of(recv, outer, extent, inner)
        for j, part in enumerate(parts):
            out[:, offs[j]:offs[j + 1], :] = part

    hap_p2p_all_gather_v = hap_p2p_all_gather_push

    def hap_p2p_reduce_scatter_direct(self, send, recv, outer, inner, extent, sizes):
        offs = np.cumsum([0] + sizes)
        parts = self._gather(np.array(self._block_of(send, outer, extent, inner), dtype=np.float64))
        self.trace.append(("p2p_reduce_scatter", tuple(sizes)))
        total = sum(parts[1:], parts[0])
        r = self.rank
        self._block_of(recv, outer, sizes[r], inner)[...] = total[:, offs[r]:offs[r + 1], :]

    hap_p2p_reduce_scatter_v = hap_p2p_reduce_scatter_direct

    def hap_p2p_all_reduce(self, send, recv, n):
        parts = self._gather(np.array(self.mem.view(send.ptr, n), dtype=np.float64))
        self.trace.append(("p2p_all_reduce", n))
        self.mem.view(recv.ptr, n)[...] = sum(parts[1:], parts[0])

    def hap_p2p_all_to_all(self, send, recv, send_off, counts, dst_off):
        flat = self.mem.view(send.ptr, send.numel)
        mine = [np.array(flat[send_off[k]:send_off[k] + counts[k]]) for k in range(self.m)]
        everyone = self._gather((mine, list(dst_off)))
        self.trace.append(("p2p_all_to_all", tuple(counts)))
        out = self.mem.view(recv.ptr, recv.numel)
        for j in range(self.m):
            chunk, offs = everyone[j][0][self.rank], everyone[j][1][self.rank]
            out[offs:offs + len(chunk)] = chunk


def step(ex) -> HostRunner:
    """Run forward + backward + update of a dry-compiled executor on the host."""
    runner = HostRunner(ex)
    runner.run(ex.ops_fwd)
    runner.run(ex.ops_bwd)
    runner.run(ex.ops_upd)
    return runner


def losses(ex) -> list:
    vals = {r: float(ex.loss_buf[r].tensor[0]) for r in ex.group.local_ranks}
    if ex.group.distributed:
        return [float(v) for v in ex.group.exchange(vals[ex.group.rank])]
    return [vals[r] for r in range(ex.m)]


_ = dist
