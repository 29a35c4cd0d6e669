"""oracle/ — TEST INFRASTRUCTURE ONLY: the parity checker for the CUDA path.

Two CPU implementations of the reference hot path, both float64:

* ``port``      — oracle/anisoq_oracle.c, a plain-C restatement of the
                  reference algorithm (each function cites file:line), built
                  into oracle/_build/liboracle.so;
* ``reference`` — the unmodified reference headers (/root/reference/proj/
                  include) compiled in place by oracle/Makefile against the
                  Eigen-subset stand-in into oracle/_ref/libanisoq_ref.so.

tests/test_oracle.py pins ``port`` against ``reference`` and the reference
tests' worked examples. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package; the product
(paper_1908_10396_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libanisoq_ref.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_szt = C.c_size_t


class OracleError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def build(force: bool = False) -> None:
    """Compile the C restatement (and oracle/_ref when the reference exists)."""
    if force or not os.path.exists(PORT_SO) or not os.path.exists(REF_SO):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            build()
        self.lib = C.CDLL(self.path)
        self.err = getattr(self.lib, self.prefix + "last_error")
        self.err.restype = C.c_char_p

    def _call(self, name, *args):
        fn = getattr(self.lib, self.prefix + name)
        st = fn(*args)
        if st:
            raise OracleError(st, self.err().decode())

    # ---- shared surface (names follow the reference) ----
    def pq_quantize(self, x, cb, M, k, sd, hp, ho, passes, threads=1):
        x = _f64(x)
        n, d = x.shape
        codes = np.zeros((n, M), np.uint32)
        extra = (C.c_int(threads),) if self.prefix == "ref_" else ()
        self._call("pq_quantize", x.ctypes.data_as(C.c_void_p), _szt(n), _szt(d),
                   _f64(cb).ctypes.data_as(C.c_void_p), _szt(M), _szt(k), _szt(sd),
                   _f64(hp).ctypes.data_as(C.c_void_p), _f64(ho).ctypes.data_as(C.c_void_p),
                   C.c_int(passes), *extra, codes.ctypes.data_as(C.c_void_p))
        return codes

    def pq_assign_pass(self, x, cb, M, k, sd, hp, ho, codes, sweep_fixed=False, threads=1):
        x = _f64(x)
        n, d = x.shape
        codes = _u32(codes).copy()
        losses = np.zeros(n, np.float64)
        extra = (C.c_int(threads),) if self.prefix == "ref_" else ()
        self._call("pq_assign_pass", x.ctypes.data_as(C.c_void_p), _szt(n), _szt(d),
                   _f64(cb).ctypes.data_as(C.c_void_p), _szt(M), _szt(k), _szt(sd),
                   _f64(hp).ctypes.data_as(C.c_void_p), _f64(ho).ctypes.data_as(C.c_void_p),
                   *extra, C.c_int(int(sweep_fixed)), codes.ctypes.data_as(C.c_void_p),
                   losses.ctypes.data_as(C.c_void_p))
        return codes, losses

    def assemble_selector_system(self, x, codes, hp, ho, M, k):
        x = _f64(x)
        n, d = x.shape
        dim = k * d
        A = np.zeros((dim, dim), np.float64)
        rhs = np.zeros(dim, np.float64)
        self._call("assemble_selector_system", x.ctypes.data_as(C.c_void_p), _szt(n),
                   _szt(d), _u32(codes).ctypes.data_as(C.c_void_p),
                   _f64(hp).ctypes.data_as(C.c_void_p), _f64(ho).ctypes.data_as(C.c_void_p),
                   _szt(M), _szt(k), A.ctypes.data_as(C.c_void_p), rhs.ctypes.data_as(C.c_void_p))
        return A, rhs

    def pq_codebook_update(self, x, codes, hp, ho, M, k, ridge=-1.0):
        x = _f64(x)
        n, d = x.shape
        out = np.zeros(k * d, np.float64)
        self._call("pq_codebook_update", x.ctypes.data_as(C.c_void_p), _szt(n), _szt(d),
                   _u32(codes).ctypes.data_as(C.c_void_p),
                   _f64(hp).ctypes.data_as(C.c_void_p), _f64(ho).ctypes.data_as(C.c_void_p),
                   _szt(M), _szt(k), C.c_double(ridge), out.ctypes.data_as(C.c_void_p))
        return out

    def train_l2_pq(self, x, M, k, max_it=100, tol=1e-6, seed=0, threads=1):
        x = _f64(x)
        n, d = x.shape
        cb = np.zeros(k * d, np.float64)
        codes = np.zeros((n, M), np.uint32)
        extra = (C.c_int(threads),) if self.prefix == "ref_" else ()
        self._call("train_l2_pq", x.ctypes.data_as(C.c_void_p), _szt(n), _szt(d), _szt(M),
                   _szt(k), C.c_int(max_it), C.c_double(tol), C.c_uint64(seed), *extra,
                   cb.ctypes.data_as(C.c_void_p), codes.ctypes.data_as(C.c_void_p))
        return cb, codes

    def train_apq(self, x, M, k, hp, ho, max_it=100, tol=1e-6, seed=0, ridge=-1.0,
                  sweep_fixed=False, warm_start=True, threads=1):
        x = _f64(x)
        n, d = x.shape
        cb = np.zeros(k * d, np.float64)
        codes = np.zeros((n, M), np.uint32)
        hist = np.zeros(max_it + 1, np.float64)
        hl = _szt(0)
        args = [x.ctypes.data_as(C.c_void_p), _szt(n), _szt(d), _szt(M), _szt(k),
                _f64(hp).ctypes.data_as(C.c_void_p), _f64(ho).ctypes.data_as(C.c_void_p),
                C.c_int(max_it), C.c_double(tol), C.c_uint64(seed), C.c_double(ridge)]
        if self.prefix == "ref_":
            args.append(C.c_int(threads))
        args += [C.c_int(int(sweep_fixed)), C.c_int(int(warm_start)),
                 cb.ctypes.data_as(C.c_void_p), codes.ctypes.data_as(C.c_void_p),
                 hist.ctypes.data_as(C.c_void_p), C.byref(hl)]
        self._call("train_apq", *args)
        return cb, codes, hist[: hl.value].copy()

    def train_avq(self, x, k, hp, ho, max_it=100, tol=1e-6, seed=0, ridge=-1.0,
                  keep_previous=False, threads=1):
        """vq.hpp:243-329 -> (codewords k x d, assignments, loss history)."""
        x = _f64(x)
        n, d = x.shape
        cw = np.zeros(k * d, np.float64)
        a = np.zeros(n, np.uint32)
        hist = np.zeros(max_it + 1, np.float64)
        hl = _szt(0)
        vp = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
        hp, ho = _f64(hp), _f64(ho)
        args = [vp(x), _szt(n), _szt(d), _szt(k), vp(hp), vp(ho), C.c_int(max_it),
                C.c_double(tol), C.c_uint64(seed), C.c_double(ridge)]
        if self.prefix == "ref_":
            args.append(C.c_int(threads))
        args += [C.c_int(1 if keep_previous else 0), vp(cw), vp(a), vp(hist), C.byref(hl)]
        self._call("train_avq", *args)
        return cw.reshape(k, d), a, hist[:hl.value].copy()

    def vq_quantize(self, x, cw, hp, ho, threads=1):
        """vq.hpp:332-343 -> assignments."""
        x, cw, hp, ho = _f64(x), _f64(cw), _f64(hp), _f64(ho)
        n, d = x.shape
        k = cw.size // d
        a = np.zeros(n, np.uint32)
        vp = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
        args = [vp(x), _szt(n), _szt(d), vp(cw), _szt(k), vp(hp), vp(ho)]
        if self.prefix == "ref_":
            args.append(C.c_int(threads))
        self._call("vq_quantize", *args, vp(a))
        return a

    def assign_point(self, x, cw, hp, ho):
        """vq.hpp:112-132 -> codeword index."""
        x, cw = _f64(x).ravel(), _f64(cw)
        out = C.c_uint32(0)
        self._call("assign_point", x.ctypes.data_as(C.c_void_p), _szt(x.size),
                   cw.ctypes.data_as(C.c_void_p), _szt(cw.size // max(x.size, 1)),
                   C.c_double(hp), C.c_double(ho), C.byref(out))
        return out.value

    def update_codeword(self, d, pts, hp, ho, ridge=-1.0):
        """vq.hpp:139-192 -> codeword (d values)."""
        pts, hp, ho = _f64(pts).ravel(), _f64(hp), _f64(ho)
        out = np.zeros(d, np.float64)
        vp = lambda v: v.ctypes.data_as(C.c_void_p)  # noqa: E731
        self._call("update_codeword", _szt(d), vp(pts), _szt(pts.size // d), vp(hp), vp(ho),
                   C.c_double(ridge), vp(out))
        return out

    def build_lut(self, q, cb, M, k, sd):
        q = _f64(q)
        lut = np.zeros(M * k, np.float64)
        self._call("build_lut", q.ctypes.data_as(C.c_void_p), _szt(q.size),
                   _f64(cb).ctypes.data_as(C.c_void_p), _szt(M), _szt(k), _szt(sd),
                   lut.ctypes.data_as(C.c_void_p))
        return lut

    def adc_search_batch(self, Q, codes, codes_k, cb, M, k, sd, topn, threads=1):
        Q = _f64(np.atleast_2d(Q))
        nq, d = Q.shape
        codes = _u32(codes)
        n = codes.shape[0]
        te = min(topn, n)
        ids = np.zeros((nq, te), np.uint32)
        sc = np.zeros((nq, te), np.float64)
        args = [Q.ctypes.data_as(C.c_void_p), _szt(nq), _szt(d), codes.ctypes.data_as(C.c_void_p),
                _szt(n), _szt(codes.shape[1] if codes.ndim == 2 else M), _szt(codes_k),
                _f64(cb).ctypes.data_as(C.c_void_p), _szt(M), _szt(k), _szt(sd), _szt(topn)]
        if self.prefix == "ref_":
            cnt = _szt(0)
            args += [C.c_int(threads), ids.ctypes.data_as(C.c_void_p),
                     sc.ctypes.data_as(C.c_void_p), C.byref(cnt)]
        else:
            args += [ids.ctypes.data_as(C.c_void_p), sc.ctypes.data_as(C.c_void_p)]
        self._call("adc_search_batch", *args)
        return ids, sc

    def rerank(self, Q, x, cand, keep, threads=1):
        Q = _f64(np.atleast_2d(Q))
        x = _f64(x)
        nq, d = Q.shape
        cand = _u32(cand)
        ncand = cand.shape[1]
        ke = min(keep, ncand)
        ids = np.zeros((nq, ke), np.uint32)
        sc = np.zeros((nq, ke), np.float64)
        args = [Q.ctypes.data_as(C.c_void_p), _szt(nq), x.ctypes.data_as(C.c_void_p),
                _szt(x.shape[0]), _szt(d), cand.ctypes.data_as(C.c_void_p), _szt(ncand),
                _szt(keep)]
        if self.prefix == "ref_":
            args.append(C.c_int(threads))
        args += [ids.ctypes.data_as(C.c_void_p), sc.ctypes.data_as(C.c_void_p)]
        self._call("rerank", *args)
        return ids, sc

    def exact_search_batch(self, Q, x, depth, threads=1):
        Q = _f64(np.atleast_2d(Q))
        x = _f64(x)
        nq, d = Q.shape
        n = x.shape[0]
        te = min(depth, n)
        ids = np.zeros((nq, te), np.uint32)
        sc = np.zeros((nq, te), np.float64)
        args = [Q.ctypes.data_as(C.c_void_p), _szt(nq), x.ctypes.data_as(C.c_void_p), _szt(n),
                _szt(d), _szt(depth)]
        if self.prefix == "ref_":
            args.append(C.c_int(threads))
        args += [ids.ctypes.data_as(C.c_void_p), sc.ctypes.data_as(C.c_void_p)]
        self._call("exact_search_batch", *args)
        return ids, sc


class Port(_Lib):
    """The C restatement (kind "port")."""

    prefix = "orc_"
    path = PORT_SO

    def row_norms(self, x):
        x = _f64(x)
        out = np.zeros(x.shape[0], np.float64)
        self.lib.orc_row_norms(x.ctypes.data_as(C.c_void_p), _szt(x.shape[0]),
                               _szt(x.shape[1]), out.ctypes.data_as(C.c_void_p))
        return out

    def threshold_weights(self, norms, d, t, policy=1):
        norms = _f64(norms)
        hp = np.zeros_like(norms)
        ho = np.zeros_like(norms)
        self._call("threshold_weights", norms.ctypes.data_as(C.c_void_p), _szt(norms.size),
                   _szt(d), C.c_double(t), C.c_int(policy), hp.ctypes.data_as(C.c_void_p),
                   ho.ctypes.data_as(C.c_void_p))
        return hp, ho

    def llt_solve(self, A, b):
        A = _f64(A)
        out = np.zeros(A.shape[0], np.float64)
        self._call("llt_solve", A.ctypes.data_as(C.c_void_p), _szt(A.shape[0]),
                   _f64(b).ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
        return out

    def pq_point_losses(self, x, cb, M, k, sd, hp, ho, codes):
        x = _f64(x)
        n, d = x.shape
        out = np.zeros(n, np.float64)
        self._call("pq_point_losses", x.ctypes.data_as(C.c_void_p), _szt(n), _szt(d),
                   _f64(cb).ctypes.data_as(C.c_void_p), _szt(M), _szt(k), _szt(sd),
                   _f64(hp).ctypes.data_as(C.c_void_p), _f64(ho).ctypes.data_as(C.c_void_p),
                   _u32(codes).ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
        return out

    def sample_distinct(self, seed, n, k):
        out = np.zeros(min(n, k), np.uintp)
        self.lib.orc_sample_distinct(C.c_uint64(seed), _szt(n), _szt(k),
                                     out.ctypes.data_as(C.c_void_p))
        return out.astype(np.int64)


class Reference(_Lib):
    """The reference headers compiled in place (kind "reference")."""

    prefix = "ref_"
    path = REF_SO

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def row_norms(self, x):
        x = _f64(x)
        out = np.zeros(x.shape[0], np.float64)
        self._call("row_norms", x.ctypes.data_as(C.c_void_p), _szt(x.shape[0]),
                   _szt(x.shape[1]), out.ctypes.data_as(C.c_void_p))
        return out

    def eta_limit(self, t, norm, d):
        out = C.c_double(0)
        self._call("eta_limit", C.c_double(t), C.c_double(norm), C.c_int(d), C.byref(out))
        return out.value

    def pq_assign_point(self, x, cur, cb, M, k, sd, hp, ho):
        out = np.zeros(M, np.uint32)
        x = _f64(x)
        self._call("pq_assign_point", x.ctypes.data_as(C.c_void_p), _szt(x.size),
                   _u32(cur).ctypes.data_as(C.c_void_p), _f64(cb).ctypes.data_as(C.c_void_p),
                   _szt(M), _szt(k), _szt(sd), C.c_double(hp), C.c_double(ho),
                   out.ctypes.data_as(C.c_void_p))
        return out

    def pq_assign_point_order(self, x, cur, cb, M, k, sd, hp, ho, order):
        out = np.zeros(M, np.uint32)
        x = _f64(x)
        order = np.ascontiguousarray(order, np.uintp)
        self._call("pq_assign_point_order", x.ctypes.data_as(C.c_void_p), _szt(x.size),
                   _u32(cur).ctypes.data_as(C.c_void_p), _f64(cb).ctypes.data_as(C.c_void_p),
                   _szt(M), _szt(k), _szt(sd), C.c_double(hp), C.c_double(ho),
                   order.ctypes.data_as(C.c_void_p), _szt(order.size),
                   out.ctypes.data_as(C.c_void_p))
        return out

    def generate_synthetic(self, kind, n, d, seed, centers=16, spread=0.25, normalize=False):
        out = np.zeros((n, d), np.float64)
        self._call("generate_synthetic", C.c_int(kind), _szt(n), _szt(d), C.c_uint64(seed),
                   _szt(centers), C.c_double(spread), C.c_int(int(normalize)),
                   out.ctypes.data_as(C.c_void_p))
        return out

    def sample_distinct(self, seed, n, k):
        out = np.zeros(min(n, k), np.uintp)
        self.lib.ref_sample_distinct(C.c_uint64(seed), _szt(n), _szt(k),
                                     out.ctypes.data_as(C.c_void_p))
        return out.astype(np.int64)
