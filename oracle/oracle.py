"""ctypes access to the CPU checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  It exposes two libraries built by
oracle/Makefile:

* ``Oracle`` — the plain-C restatement (oracle/covap_oracle.c), fp32 and fp64;
* ``Ref``    — the reference library itself, compiled from
  /root/reference/proj/src (+ oracle/ref_shim.cpp), when it was built.

Neither is ever on the product path (paper_2311_04499_b200/).
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libcovap_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcovap_ref.so")
REF_SRC = "/root/reference/proj"

_u8 = ctypes.POINTER(ctypes.c_uint8)
_u32 = ctypes.POINTER(ctypes.c_uint32)
_u64 = ctypes.POINTER(ctypes.c_uint64)
_f32 = ctypes.POINTER(ctypes.c_float)
_f64 = ctypes.POINTER(ctypes.c_double)
_sz = ctypes.c_size_t


def build(ref=True):
    """make -C oracle (restatement always; the reference only where its
    sources exist, i.e. in the build container)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REF_SRC):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _p(a, t):
    return a.ctypes.data_as(t)


def _arr(x, dtype):
    return np.ascontiguousarray(np.asarray(x, dtype=dtype))


class OracleError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where}: status {code}")
        self.code = code


def _ck(code, where):
    if code:
        raise OracleError(code, where)


class OcFilter(ctypes.Structure):
    """oc_filter (covap_oracle.h)."""
    _fields_ = [("kind", ctypes.c_int), ("interval", ctypes.c_uint32), ("rule", ctypes.c_int),
                ("k_fraction", ctypes.c_double), ("seed", ctypes.c_uint64)]


class Oracle:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        self.d = ctypes.CDLL(path)
        self.d.oc_stream_key.restype = ctypes.c_uint64
        self.d.oc_stream_key.argtypes = [ctypes.c_uint64] * 3
        self.d.oc_generate_f32.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.c_uint64, _f32]
        self.d.oc_generate_f64.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.c_uint64, _f64]
        self.d.oc_ef_coefficient.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_uint64,
                                             ctypes.c_double, _f64]
        self.d.oc_ccr.argtypes = [ctypes.c_double, ctypes.c_double, _f64]
        self.d.oc_choose_interval.argtypes = [ctypes.c_double, _u32]
        self.d.oc_compress_f32.argtypes = [_f32, _f32, _sz, _u64, _u64, _u8, ctypes.c_int,
                                           ctypes.c_float, _f32, _u64]
        self.d.oc_compress_f64.argtypes = [_f64, _f64, _sz, _u64, _u64, _u8, ctypes.c_int,
                                           ctypes.c_double, _f64, _u64]
        self.d.oc_profile_ccr.argtypes = [_f64, _f64, _sz, _sz, ctypes.c_double, _f64, _f64, _f64,
                                          _u32]

    # planner -------------------------------------------------------------
    def allocate_buckets(self, layer_numel, cap_bytes, bpp=None):
        ln = _arr(layer_numel, np.uint64)
        bp = None if bpp is None else _p(_arr(bpp, np.uint32), _u32)
        out = np.zeros(len(ln) + 1, np.uint64)
        first = np.zeros(len(ln) + 1, np.uint64)
        nb = _sz()
        _ck(self.d.oc_allocate_buckets(_p(ln, _u64), bp, _sz(len(ln)), ctypes.c_uint64(cap_bytes),
                                       _p(out, _u64), _p(first, _u64), _sz(len(out)),
                                       ctypes.byref(nb)), "allocate_buckets")
        return out[:nb.value].tolist(), first[:nb.value].tolist()

    def median_twice(self, bucket_numel):
        b = _arr(bucket_numel, np.uint64)
        t = ctypes.c_uint64()
        _ck(self.d.oc_median_twice(_p(b, _u64), _sz(len(b)), ctypes.byref(t)), "median")
        return t.value

    def effective_tensors(self, bucket_numel, interval, shard):
        b = _arr(bucket_numel, np.uint64)
        cap = int(sum(min(interval, 1 << 20) for _ in b)) + len(b) + 1
        tb, tbeg, tend = (np.zeros(cap, np.uint64) for _ in range(3))
        nt = _sz()
        _ck(self.d.oc_effective_tensors(_p(b, _u64), _sz(len(b)), ctypes.c_uint32(interval),
                                        ctypes.c_int(shard), _p(tb, _u64), _p(tbeg, _u64),
                                        _p(tend, _u64), _sz(cap), ctypes.byref(nt)),
            "effective_tensors")
        n = nt.value
        return [(int(tb[i]), int(tbeg[i]), int(tend[i])) for i in range(n)]

    def plan(self, layer_numel, cap_bytes, interval, shard=None):
        """train()'s plan: allocate, shard when K > 1 (trainer.cpp:266-271)."""
        buckets, first = self.allocate_buckets(layer_numel, cap_bytes)
        if shard is None:
            shard = interval > 1
        return buckets, self.effective_tensors(buckets, interval, int(shard))

    def select(self, step, interval, count, rule=0):
        keep = np.zeros(max(count, 1), np.uint8)
        _ck(self.d.oc_select(ctypes.c_uint64(step), ctypes.c_uint32(interval), _sz(count),
                             ctypes.c_int(rule), _p(keep, _u8)), "select")
        return keep[:count]

    def ef_coefficient(self, step, init=0.3, ascend=100, rng=0.1):
        c = ctypes.c_double()
        _ck(self.d.oc_ef_coefficient(step, init, ascend, rng, ctypes.byref(c)), "ef")
        return c.value

    # compress / decompress ------------------------------------------------
    def compress(self, g, r, tensors, keep, ef_enabled, coeff):
        """Flat covap_compress; r updated in place; returns payload."""
        dt = g.dtype
        tb = _arr([t[1] for t in tensors], np.uint64)
        te = _arr([t[2] for t in tensors], np.uint64)
        kp = _arr(keep, np.uint8)
        payload = np.zeros(max(int(sum(t[2] - t[1] for t, k in zip(tensors, kp) if k)), 1), dt)
        n = ctypes.c_uint64()
        if dt == np.float32:
            _ck(self.d.oc_compress_f32(_p(g, _f32), _p(r, _f32), _sz(len(tensors)), _p(tb, _u64),
                                       _p(te, _u64), _p(kp, _u8), int(ef_enabled),
                                       np.float32(coeff).item(), _p(payload, _f32),
                                       ctypes.byref(n)), "compress")
        else:
            _ck(self.d.oc_compress_f64(_p(g, _f64), _p(r, _f64), _sz(len(tensors)), _p(tb, _u64),
                                       _p(te, _u64), _p(kp, _u8), int(ef_enabled), float(coeff),
                                       _p(payload, _f64), ctypes.byref(n)), "compress")
        return payload[:n.value]

    def decompress(self, payload, tensors, keep, total, dtype):
        tb = _arr([t[1] for t in tensors], np.uint64)
        te = _arr([t[2] for t in tensors], np.uint64)
        kp = _arr(keep, np.uint8)
        out = np.empty(total, dtype)
        payload = np.ascontiguousarray(payload, dtype)
        fn = self.d.oc_decompress_f32 if dtype == np.float32 else self.d.oc_decompress_f64
        pt = _f32 if dtype == np.float32 else _f64
        _ck(fn(_p(payload, pt), _sz(len(tensors)), _p(tb, _u64), _p(te, _u64), _p(kp, _u8),
               _p(out, pt)), "decompress")
        return out

    def allreduce_mean(self, per_worker):
        pw = np.ascontiguousarray(per_worker)
        P, n = pw.shape
        out = np.empty(n, pw.dtype)
        if pw.dtype == np.float32:
            _ck(self.d.oc_allreduce_mean_f32(_p(pw, _f32), _sz(P), _sz(n), _p(out, _f32)), "mean")
        else:
            _ck(self.d.oc_allreduce_mean_f64(_p(pw, _f64), _sz(P), _sz(n), _p(out, _f64)), "mean")
        return out

    # CCR -----------------------------------------------------------------
    def ccr(self, comm, comp):
        c = ctypes.c_double()
        _ck(self.d.oc_ccr(comm, comp, ctypes.byref(c)), "ccr")
        return c.value

    def choose_interval(self, c):
        k = ctypes.c_uint32()
        _ck(self.d.oc_choose_interval(c, ctypes.byref(k)), "choose_interval")
        return k.value

    def profile_ccr(self, starts, ends, comp_ms):
        s = _arr(starts, np.float64)
        e = _arr(ends, np.float64)
        W, C = s.shape
        naive = np.zeros(W)
        a, c, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint32()
        _ck(self.d.oc_profile_ccr(_p(s, _f64), _p(e, _f64), W, C, comp_ms, ctypes.byref(a),
                                  _p(naive, _f64), ctypes.byref(c), ctypes.byref(k)), "profile")
        return a.value, naive.tolist(), c.value, k.value

    # baseline compressors / error feedback ---------------
    def sparsifier_k(self, d, k_fraction):
        k = ctypes.c_uint64()
        self.d.oc_sparsifier_k.argtypes = [ctypes.c_uint64, ctypes.c_double, _u64]
        _ck(self.d.oc_sparsifier_k(d, k_fraction, ctypes.byref(k)), "sparsifier_k")
        return k.value

    def half_bits(self, v):
        self.d.oc_half_bits_from_float.restype = ctypes.c_uint16
        self.d.oc_half_bits_from_float.argtypes = [ctypes.c_float, ctypes.POINTER(ctypes.c_int)]
        sat = ctypes.c_int(0)
        h = self.d.oc_half_bits_from_float(float(v), ctypes.byref(sat))
        return h, bool(sat.value)

    def float_from_half(self, h):
        self.d.oc_float_from_half_bits.restype = ctypes.c_float
        self.d.oc_float_from_half_bits.argtypes = [ctypes.c_uint16]
        return self.d.oc_float_from_half_bits(int(h))

    def fp16_roundtrip(self, x):
        x = np.ascontiguousarray(x)
        out = np.empty_like(x)
        sat = ctypes.c_uint64(0)
        if x.dtype == np.float32:
            self.d.oc_fp16_roundtrip_f32.argtypes = [_f32, ctypes.c_uint64, _f32, _u64]
            self.d.oc_fp16_roundtrip_f32(_p(x, _f32), len(x), _p(out, _f32), ctypes.byref(sat))
        else:
            self.d.oc_fp16_roundtrip_f64.argtypes = [_f64, ctypes.c_uint64, _f64, _u64]
            self.d.oc_fp16_roundtrip_f64(_p(x, _f64), len(x), _p(out, _f64), ctypes.byref(sat))
        return out, sat.value

    def topk(self, x, k_fraction):
        """(indices in the reference's order, values)."""
        x = np.ascontiguousarray(x)
        idx = np.zeros(max(len(x), 1), np.uint64)
        k = ctypes.c_uint64()
        if x.dtype == np.float32:
            self.d.oc_topk_f32.argtypes = [_f32, ctypes.c_uint64, ctypes.c_double, _u64, _u64]
            _ck(self.d.oc_topk_f32(_p(x, _f32), len(x), k_fraction, _p(idx, _u64),
                                   ctypes.byref(k)), "topk")
        else:
            self.d.oc_topk_f64.argtypes = [_f64, ctypes.c_uint64, ctypes.c_double, _u64, _u64]
            _ck(self.d.oc_topk_f64(_p(x, _f64), len(x), k_fraction, _p(idx, _u64),
                                   ctypes.byref(k)), "topk")
        i = idx[:k.value].copy()
        return i, x[i]

    def randomk(self, d, k_fraction, seed):
        idx = np.zeros(max(d, 1), np.uint64)
        k = ctypes.c_uint64()
        self.d.oc_randomk.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_uint64, _u64, _u64]
        _ck(self.d.oc_randomk(d, k_fraction, ctypes.c_uint64(seed), _p(idx, _u64),
                              ctypes.byref(k)), "randomk")
        return idx[:k.value].copy()

    def mix_seed(self, seed, tag):
        self.d.oc_mix_seed.restype = ctypes.c_uint64
        self.d.oc_mix_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        return self.d.oc_mix_seed(seed, tag)

    def feedback_step(self, kind, num_steps, g, r, tensors, ef_enabled, coeff, interval=1,
                      rule=0, k_fraction=0.01, seed=0):
        """ErrorFeedback::step; r updated in place; returns (kept, transmitted, saturations)."""
        f = OcFilter(kind, interval, rule, k_fraction, seed)
        tb = _arr([t[1] for t in tensors], np.uint64)
        te = _arr([t[2] for t in tensors], np.uint64)
        kept = np.zeros_like(g)
        sent, sat = ctypes.c_uint64(), ctypes.c_uint64(0)
        if g.dtype == np.float32:
            fn, pt, c = self.d.oc_feedback_step_f32, _f32, ctypes.c_float(np.float32(coeff).item())
        else:
            fn, pt, c = self.d.oc_feedback_step_f64, _f64, ctypes.c_double(float(coeff))
        fn.argtypes = [ctypes.POINTER(OcFilter), ctypes.c_uint64, pt, pt, _sz, _u64, _u64,
                       ctypes.c_int, type(c), pt, _u64, _u64]
        _ck(fn(ctypes.byref(f), num_steps, _p(g, pt), _p(r, pt), len(tensors), _p(tb, _u64),
               _p(te, _u64), int(ef_enabled), c, _p(kept, pt), ctypes.byref(sent),
               ctypes.byref(sat)), "feedback_step")
        return kept, sent.value, sat.value

    # inputs --------------------------------------------------------------
    def stream_key(self, seed, rank, step):
        return self.d.oc_stream_key(seed, rank, step)

    def generate(self, key, n, kind=0, begin=0, dtype=np.float32):
        out = np.empty(n, dtype)
        if dtype == np.float32:
            self.d.oc_generate_f32(key, kind, begin, n, _p(out, _f32))
        else:
            self.d.oc_generate_f64(key, kind, begin, n, _p(out, _f64))
        return out


class Ref:
    """The reference library compiled from its own sources (oracle/_ref)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REF_SRC):
                build(ref=True)
            else:
                raise FileNotFoundError(path)
        self.d = ctypes.CDLL(path)
        d = self.d
        d.ref_plan.argtypes = [_u64, _u32, _sz, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, _u64,
                               _sz, ctypes.POINTER(_sz), _u64, _u64, _u64, _u64, _sz,
                               ctypes.POINTER(_sz)]
        d.ref_select.argtypes = [ctypes.c_uint64, ctypes.c_uint32, _sz, ctypes.c_int, _u64,
                                 ctypes.POINTER(_sz)]
        d.ref_ef_coefficient.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_uint64, ctypes.c_double, _f64]
        d.ref_compress.argtypes = [_f64, _u64, _sz, _f64, _u64, ctypes.c_uint32, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_double,
                                   _f64, _u64, ctypes.POINTER(_sz)]
        d.ref_decompress.argtypes = [_f64, _u64, _sz, _u64, _sz, _f64]
        d.ref_allreduce_mean.argtypes = [_f64, _sz, _sz, _f64]
        d.ref_ccr.argtypes = [ctypes.c_double, ctypes.c_double, _f64]
        d.ref_choose_interval.argtypes = [ctypes.c_double, _u32]
        d.ref_profile_ccr.argtypes = [_f64, _f64, _sz, ctypes.c_uint32, _sz, ctypes.c_double, _f64,
                                      _f64, _f64, _u32]
        d.ref_session_create.restype = ctypes.c_void_p
        d.ref_session_create.argtypes = [_u64, _sz, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                         ctypes.c_double]
        d.ref_session_destroy.argtypes = [ctypes.c_void_p]
        d.ref_session_step.argtypes = [ctypes.c_void_p, _f64, _f64, _f64, _f64]

    def plan(self, layer_numel, cap_bytes, interval, shard=None, bpp=None):
        ln = _arr(layer_numel, np.uint64)
        if shard is None:
            shard = interval > 1
        bp = None if bpp is None else _p(_arr(bpp, np.uint32), _u32)
        nbmax = len(ln) + 1
        ntmax = nbmax * max(1, min(interval, 4096)) + 1
        bn = np.zeros(nbmax, np.uint64)
        tb, tbeg, tend = (np.zeros(ntmax, np.uint64) for _ in range(3))
        nb, nt, tw = _sz(), _sz(), ctypes.c_uint64()
        _ck(self.d.ref_plan(_p(ln, _u64), bp, _sz(len(ln)), ctypes.c_uint64(cap_bytes),
                            ctypes.c_uint32(interval), int(shard), _p(bn, _u64), _sz(nbmax),
                            ctypes.byref(nb), ctypes.byref(tw), _p(tb, _u64), _p(tbeg, _u64),
                            _p(tend, _u64), _sz(ntmax), ctypes.byref(nt)), "ref_plan")
        tensors = [(int(tb[i]), int(tbeg[i]), int(tend[i])) for i in range(nt.value)]
        return bn[:nb.value].tolist(), tw.value, tensors

    def select(self, step, interval, count, rule=0):
        out = np.zeros(max(count, 1), np.uint64)
        n = _sz()
        _ck(self.d.ref_select(step, interval, count, rule, _p(out, _u64), ctypes.byref(n)),
            "ref_select")
        return out[:n.value].tolist()

    def ef_coefficient(self, step, enabled=1, init=0.3, ascend=100, rng=0.1):
        c = ctypes.c_double()
        _ck(self.d.ref_ef_coefficient(step, enabled, init, ascend, rng, ctypes.byref(c)), "ref_ef")
        return c.value

    def compress(self, g, numels, residual, num_steps, interval, rule=0, ef=(1, 0.3, 100, 0.1)):
        """Returns payload, selected, num_steps'; residual updated in place."""
        nv = _arr(numels, np.uint64)
        g = np.ascontiguousarray(g, np.float64)
        payload = np.zeros(max(len(g), 1), np.float64)
        sel = np.zeros(len(nv) + 1, np.uint64)
        ns = ctypes.c_uint64(num_steps)
        n = _sz()
        _ck(self.d.ref_compress(_p(g, _f64), _p(nv, _u64), _sz(len(nv)), _p(residual, _f64),
                                ctypes.byref(ns), interval, rule, int(ef[0]), float(ef[1]),
                                int(ef[2]), float(ef[3]), _p(payload, _f64), _p(sel, _u64),
                                ctypes.byref(n)), "ref_compress")
        selected = sel[:n.value].tolist()
        return payload[:int(sum(numels[t] for t in selected))], selected, ns.value

    def decompress(self, payload, selected, numels):
        nv = _arr(numels, np.uint64)
        s = _arr(selected, np.uint64) if len(selected) else np.zeros(1, np.uint64)
        out = np.empty(int(sum(numels)), np.float64)
        pl = np.ascontiguousarray(payload, np.float64) if len(payload) else np.zeros(1)
        _ck(self.d.ref_decompress(_p(pl, _f64), _p(s, _u64), _sz(len(selected)), _p(nv, _u64),
                                  _sz(len(nv)), _p(out, _f64)), "ref_decompress")
        return out

    def allreduce_mean(self, per_worker):
        pw = np.ascontiguousarray(per_worker, np.float64)
        P, n = pw.shape
        out = np.empty(n)
        _ck(self.d.ref_allreduce_mean(_p(pw, _f64), P, n, _p(out, _f64)), "ref_mean")
        return out

    def ccr(self, comm, comp):
        c = ctypes.c_double()
        _ck(self.d.ref_ccr(comm, comp, ctypes.byref(c)), "ref_ccr")
        return c.value

    def choose_interval(self, c):
        k = ctypes.c_uint32()
        _ck(self.d.ref_choose_interval(c, ctypes.byref(k)), "ref_choose")
        return k.value

    def overlap_schedule(self, before, comp, compress, comm, communicated):
        n = len(comp)
        c = _arr(comp, np.float64)
        cm = _arr(comm, np.float64)
        cp = None if compress is None else _p(_arr(compress, np.float64), _f64)
        sent = None if communicated is None else _p(_arr(communicated, np.uint8), _u8)
        tot, se, un = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        cs, ce = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        ct = np.zeros(max(n, 1), np.int64)
        ba, bm = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1))
        nc, nb = _sz(), _sz()
        i64 = ctypes.POINTER(ctypes.c_int64)
        self.d.ref_overlap_schedule.argtypes = [ctypes.c_double, _f64, _f64, _f64, _u8, _sz, _f64, _f64,
                                                _f64, _f64, _f64, i64, ctypes.POINTER(_sz), i64, _f64,
                                                ctypes.POINTER(_sz)]
        _ck(self.d.ref_overlap_schedule(before, _p(c, _f64), cp, _p(cm, _f64), sent, n,
                                        ctypes.byref(tot), ctypes.byref(se), ctypes.byref(un),
                                        _p(cs, _f64), _p(ce, _f64), _p(ct, i64), ctypes.byref(nc),
                                        _p(ba, i64), _p(bm, _f64), ctypes.byref(nb)), "ref_overlap")
        k, b = nc.value, nb.value
        return {"total": tot.value, "stream_end": se.value, "unoverlapped": un.value,
                "comm_start": cs[:k].tolist(), "comm_end": ce[:k].tolist(),
                "comm_tensor": ct[:k].tolist(), "bubble_after": ba[:b].tolist(),
                "bubble_ms": bm[:b].tolist()}

    # baseline compressors / error feedback (compress.cpp:107-344) ---------
    def topk(self, x, k_fraction):
        x = np.ascontiguousarray(x, np.float64)
        idx = np.zeros(max(len(x), 1), np.uint64)
        val = np.zeros(max(len(x), 1))
        k = _sz()
        self.d.ref_topk.argtypes = [_f64, _sz, ctypes.c_double, _u64, _f64, ctypes.POINTER(_sz)]
        _ck(self.d.ref_topk(_p(x, _f64), len(x), k_fraction, _p(idx, _u64), _p(val, _f64),
                            ctypes.byref(k)), "ref_topk")
        return idx[:k.value].copy(), val[:k.value].copy()

    def randomk(self, x, k_fraction, seed):
        x = np.ascontiguousarray(x, np.float64)
        idx = np.zeros(max(len(x), 1), np.uint64)
        val = np.zeros(max(len(x), 1))
        k = _sz()
        self.d.ref_randomk.argtypes = [_f64, _sz, ctypes.c_double, ctypes.c_uint64, _u64, _f64,
                                       ctypes.POINTER(_sz)]
        _ck(self.d.ref_randomk(_p(x, _f64), len(x), k_fraction, ctypes.c_uint64(seed),
                               _p(idx, _u64), _p(val, _f64), ctypes.byref(k)), "ref_randomk")
        return idx[:k.value].copy(), val[:k.value].copy()

    def fp16_roundtrip(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        sat = ctypes.c_uint64()
        self.d.ref_fp16_roundtrip.argtypes = [_f64, _sz, _f64, _u64]
        _ck(self.d.ref_fp16_roundtrip(_p(x, _f64), len(x), _p(out, _f64), ctypes.byref(sat)),
            "ref_fp16")
        return out, sat.value

    def half_bits(self, v):
        self.d.ref_half_bits.restype = ctypes.c_uint16
        self.d.ref_half_bits.argtypes = [ctypes.c_float, ctypes.POINTER(ctypes.c_int)]
        sat = ctypes.c_int(0)
        h = self.d.ref_half_bits(float(v), ctypes.byref(sat))
        return h, bool(sat.value)

    def float_from_half(self, h):
        self.d.ref_float_from_half.restype = ctypes.c_float
        self.d.ref_float_from_half.argtypes = [ctypes.c_uint16]
        return self.d.ref_float_from_half(int(h))

    def profile_ccr(self, starts, ends, comp_ms, expected=None):
        s = _arr(starts, np.float64)
        e = _arr(ends, np.float64)
        W, C = s.shape
        naive = np.zeros(max(W, 1))
        a, c, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint32()
        _ck(self.d.ref_profile_ccr(_p(s, _f64), _p(e, _f64), W, W if expected is None else expected,
                                   C, comp_ms, ctypes.byref(a), _p(naive, _f64), ctypes.byref(c),
                                   ctypes.byref(k)), "ref_profile")
        return a.value, naive[:W].tolist(), c.value, k.value


class RefSession:
    """The reference's per-step COVAP sync sequence (trainer.cpp:365-386)."""

    def __init__(self, ref, numels, P, interval, rule=0, ef=(1, 0.3, 100, 0.1)):
        self.ref = ref
        self.numels = list(numels)
        self.d = int(sum(numels))
        self.P = P
        nv = _arr(numels, np.uint64)
        self.h = ref.d.ref_session_create(_p(nv, _u64), len(nv), P, interval, rule, int(ef[0]),
                                          float(ef[1]), int(ef[2]), float(ef[3]))

    def step(self, grads, want_residual=False):
        g = np.ascontiguousarray(grads, np.float64).reshape(self.P, self.d)
        upd = np.empty(self.d)
        res = np.empty(self.d) if want_residual else None
        sec = ctypes.c_double()
        _ck(self.ref.d.ref_session_step(self.h, _p(g, _f64), _p(upd, _f64),
                                        None if res is None else _p(res, _f64),
                                        ctypes.byref(sec)), "ref_session_step")
        return upd, res, sec.value

    def close(self):
        if self.h:
            self.ref.d.ref_session_destroy(self.h)
            self.h = None


class RefFeedback:
    """The reference's ErrorFeedback around one GradientFilter
    (compress.cpp:241-344).  kind: 0 identity, 1 covap, 2 topk, 3 randomk, 4 fp16."""

    def __init__(self, ref, numels, kind, interval=1, rule=0, k_fraction=0.01, seed=0,
                 ef=(1, 0.3, 100, 0.1)):
        self.ref = ref
        self.numels = list(numels)
        self.d = int(sum(numels))
        nv = _arr(numels, np.uint64)
        f = ref.d
        f.ref_feedback_create.restype = ctypes.c_void_p
        f.ref_feedback_create.argtypes = [_u64, _sz, ctypes.c_int, ctypes.c_uint32, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_uint64, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_uint64, ctypes.c_double]
        f.ref_feedback_destroy.argtypes = [ctypes.c_void_p]
        f.ref_feedback_step.argtypes = [ctypes.c_void_p, _f64, _f64, _f64, _u64, _f64]
        self.h = f.ref_feedback_create(_p(nv, _u64), len(nv), kind, interval, rule, k_fraction,
                                       ctypes.c_uint64(seed), int(ef[0]), float(ef[1]),
                                       int(ef[2]), float(ef[3]))

    def step(self, g):
        """Returns (kept, residual, transmitted elements, seconds)."""
        g = np.ascontiguousarray(g, np.float64)
        kept, res = np.empty(self.d), np.empty(self.d)
        sent, sec = ctypes.c_uint64(), ctypes.c_double()
        _ck(self.ref.d.ref_feedback_step(self.h, _p(g, _f64), _p(kept, _f64), _p(res, _f64),
                                         ctypes.byref(sent), ctypes.byref(sec)), "ref_feedback")
        return kept, res, sent.value, sec.value

    def close(self):
        if self.h:
            self.ref.d.ref_feedback_destroy(self.h)
            self.h = None
