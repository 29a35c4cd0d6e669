"""Python mirror of the reference `anisoq` hot-path API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/anisoq (pq.hpp, index.hpp, geometry.hpp,
error.hpp); every call runs on the B200 through libanisoq_b200.so. Types are
thin numpy holders with the reference's field names:

    Dataset(values n x d, norms)            dataset.hpp:41-51
    ProductCodebook(M, k, sub_dimension, dictionaries)   pq.hpp:39-52
    CodeMatrix(n, M, k, codes n x M uint32)  pq.hpp:55-67
    AnisotropicWeights(h_parallel, h_perpendicular)      geometry.hpp:119-145
    TrainConfig                              vq.hpp:55-69
    Hit / SearchResult                       index.hpp:46-54

Per-point weights may be given as a list/array of AnisotropicWeights (the
reference's std::span<const AnisotropicWeights>), as a single
AnisotropicWeights (uniform), or as ThresholdWeights(T) (the CLI's
resolve_weights, anisoq_main.cpp:108-142, computed on the device).
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib

_L = _lib.load()

# ---- errors (error.hpp:25-55) ---------------------------------------------


class Error(RuntimeError):
    """anisoq::Error; `error_class` is "validation" or "runtime"."""

    status = 0

    def __init__(self, what: str):
        super().__init__(what)
        self.error_class = "runtime" if _L.aq_error_class(self.status) else "validation"


def _mk(name, status):
    return type(name, (Error,), {"status": status})


InvalidArgument = _mk("InvalidArgument", 1)
ZeroNormDatapoint = _mk("ZeroNormDatapoint", 2)
InvalidThreshold = _mk("InvalidThreshold", 3)
EmptyDataset = _mk("EmptyDataset", 4)
EmptyIndex = _mk("EmptyIndex", 5)
DimensionMismatch = _mk("DimensionMismatch", 6)
DimensionNotDivisible = _mk("DimensionNotDivisible", 7)
CodeOutOfRange = _mk("CodeOutOfRange", 8)
MalformedFile = _mk("MalformedFile", 9)
InsufficientData = _mk("InsufficientData", 10)
GroundTruthMismatch = _mk("GroundTruthMismatch", 11)
QuadratureFailure = _mk("QuadratureFailure", 12)
SingularSystem = _mk("SingularSystem", 13)
DeviceError = _mk("DeviceError", 100)
Unsupported = _mk("Unsupported", 101)

_BY_STATUS = {c.status: c for c in (
    InvalidArgument, ZeroNormDatapoint, InvalidThreshold, EmptyDataset, EmptyIndex,
    DimensionMismatch, DimensionNotDivisible, CodeOutOfRange, MalformedFile,
    InsufficientData, GroundTruthMismatch, QuadratureFailure, SingularSystem,
    DeviceError, Unsupported)}


def _check(st: int) -> None:
    if st:
        raise _BY_STATUS.get(st, Error)(_L.aq_last_error().decode())


# ---- types -----------------------------------------------------------------


@dataclass
class AnisotropicWeights:
    h_parallel: float = 1.0
    h_perpendicular: float = 1.0

    @property
    def eta(self) -> float:
        return (self.h_parallel / self.h_perpendicular if self.h_perpendicular > 0
                else math.inf)

    def is_isotropic(self) -> bool:
        return self.h_parallel == self.h_perpendicular

    @staticmethod
    def from_h(h_parallel: float, h_perpendicular: float) -> "AnisotropicWeights":
        if not (h_parallel >= 0.0 and h_perpendicular >= 0.0 and math.isfinite(h_parallel)
                and math.isfinite(h_perpendicular)):
            raise InvalidArgument("InvalidArgument: h coefficients must be finite and >= 0")
        return AnisotropicWeights(float(h_parallel), float(h_perpendicular))

    @staticmethod
    def from_eta(eta: float) -> "AnisotropicWeights":
        if not eta >= 0.0:
            raise InvalidArgument("InvalidArgument: eta must be >= 0")
        return AnisotropicWeights.from_h(eta, 1.0)

    @staticmethod
    def isotropic(h: float = 1.0) -> "AnisotropicWeights":
        return AnisotropicWeights.from_h(h, h)


@dataclass
class ThresholdWeights:
    """h_par = eta_limit(T, |x_i|, d), h_perp = 1 per point (geometry.hpp:395-402).

    policy "throw" reproduces the reference (InvalidThreshold when |x_i| <= T);
    "parallel_only" uses eta = inf -> (h_par, h_perp) = (1, 0)."""

    threshold: float = 0.2
    policy: str = "throw"


def eta_limit(threshold: float, norm: float, d: int) -> float:
    """geometry.hpp:395-402 (host scalar helper)."""
    if not norm > 0.0:
        raise InvalidArgument("InvalidArgument: norm must be positive")
    if not threshold >= 0.0 or threshold >= norm:
        raise InvalidThreshold("InvalidThreshold: need 0 <= T < norm")
    if d < 2:
        raise InvalidArgument("InvalidArgument: eta_limit needs d >= 2")
    rho = (threshold / norm) * (threshold / norm)
    return float(d - 1) * rho / (1.0 - rho)


@dataclass
class Dataset:
    values: np.ndarray  # n x d: float32 when float32-exact, else float64
    normalized: bool = False

    def __post_init__(self):
        v = np.asarray(self.values)
        if v.ndim != 2:
            raise InvalidArgument("InvalidArgument: dataset must be n x d")
        if v.size and not np.all(np.isfinite(v)):  # make_dataset (dataset.hpp:100-108)
            row = int(np.nonzero(~np.isfinite(v))[0][0])
            raise MalformedFile(f"MalformedFile: non-finite value at row {row}")
        if v.dtype != np.float32:
            # float32 storage when exact (fvecs / generate_synthetic data,
            # dataset.hpp:146-151, 288: the fast kernels); float64 otherwise
            # (e.g. unit_normalize output), which runs the generic kernels
            f = v.astype(np.float32)
            v64 = np.asarray(v, np.float64)
            v = f if np.array_equal(f.astype(np.float64), v64) else v64
        self.values = np.ascontiguousarray(v)

    @property
    def f64(self) -> bool:
        return self.values.dtype == np.float64

    @property
    def n(self) -> int:
        return self.values.shape[0]

    @property
    def d(self) -> int:
        return self.values.shape[1]

    def row(self, i: int) -> np.ndarray:
        return self.values[i].astype(np.float64)


@dataclass
class ProductCodebook:
    M: int = 0
    k: int = 0
    sub_dimension: int = 0
    dictionaries: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def __post_init__(self):
        self.dictionaries = np.ascontiguousarray(self.dictionaries, dtype=np.float64).ravel()

    def dim(self) -> int:
        return self.M * self.sub_dimension

    def codeword(self, m: int, j: int) -> np.ndarray:
        o = (m * self.k + j) * self.sub_dimension
        return self.dictionaries[o:o + self.sub_dimension]


@dataclass
class CodeMatrix:
    n: int = 0
    M: int = 0
    k: int = 0
    codes: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.uint32))

    def __post_init__(self):
        self.codes = np.ascontiguousarray(self.codes, dtype=np.uint32).reshape(self.n, self.M)

    def row(self, i: int) -> np.ndarray:
        return self.codes[i]


@dataclass
class TrainConfig:
    max_iterations: int = 100
    relative_tolerance: float = 1e-6
    seed: int = 0
    empty_partition_policy: str = "reseed_highest_loss"
    ridge: float = -1.0
    threads: int = 1
    sweep_to_fixed_point: bool = False

    def c(self) -> _lib.aq_train_config:
        return _lib.aq_train_config(
            self.max_iterations, self.relative_tolerance, self.seed,
            0 if self.empty_partition_policy == "reseed_highest_loss" else 1,
            self.ridge, self.threads, int(self.sweep_to_fixed_point))


@dataclass
class Hit:
    index: int
    score: float


@dataclass
class SearchResult:
    hits: list


@dataclass
class LookupTable:
    M: int
    k: int
    partials: np.ndarray

    def at(self, m: int, j: int) -> float:
        return float(self.partials[m * self.k + j])


# ---- session -----------------------------------------------------------------


class Session:
    """One CUDA device + stream; owns device-resident objects."""

    _default: dict[int, "Session"] = {}

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(_L.aq_session_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Session":
        if device not in cls._default:
            cls._default[device] = Session(device)
        return cls._default[device]

    @property
    def stream(self) -> int:
        return _L.aq_session_stream(self.h) or 0

    def sync(self) -> None:
        _check(_L.aq_session_sync(self.h))

    @property
    def launches(self) -> int:
        return int(_L.aq_session_launches(self.h))

    def close(self) -> None:
        if self.h:
            _L.aq_session_destroy(self.h)
            self.h = None

    # device-resident objects
    def upload_dataset(self, values: np.ndarray) -> "DeviceDataset":
        ds = values if isinstance(values, Dataset) else Dataset(values)
        h = C.c_void_p()
        up = _L.aq_dataset_upload_f64 if ds.f64 else _L.aq_dataset_upload
        _check(up(self.h, ds.values.ctypes.data, ds.n, ds.d, C.byref(h)))
        return DeviceDataset(self, h, ds.n, ds.d)

    def wrap_device_rows(self, ptr: int, n: int, d: int) -> "DeviceDataset":
        h = C.c_void_p()
        _check(_L.aq_dataset_wrap_device(self.h, ptr, n, d, C.byref(h)))
        return DeviceDataset(self, h, n, d)

    def upload_codebook(self, cb: ProductCodebook) -> "DeviceCodebook":
        h = C.c_void_p()
        _check(_L.aq_codebook_upload(self.h, cb.dictionaries.ctypes.data, cb.M, cb.k,
                                     cb.sub_dimension, C.byref(h)))
        return DeviceCodebook(self, h, cb.M, cb.k, cb.sub_dimension)

    def alloc_codes(self, n: int, M: int, k: int) -> "DeviceCodes":
        h = C.c_void_p()
        _check(_L.aq_codes_alloc(self.h, n, M, k, C.byref(h)))
        return DeviceCodes(self, h, n, M, k)

    def upload_codes(self, cm: CodeMatrix) -> "DeviceCodes":
        h = C.c_void_p()
        _check(_L.aq_codes_upload(self.h, cm.codes.ctypes.data, cm.n, cm.M, cm.k, C.byref(h)))
        return DeviceCodes(self, h, cm.n, cm.M, cm.k)

    def upload_packed_codes(self, packed: np.ndarray, n: int, M: int, k: int) -> "DeviceCodes":
        packed = np.ascontiguousarray(packed, np.uint8)
        h = C.c_void_p()
        _check(_L.aq_codes_upload_packed(self.h, packed.ctypes.data, n, M, k, C.byref(h)))
        return DeviceCodes(self, h, n, M, k)


class _Handle:
    _free = None

    def free(self):
        if getattr(self, "h", None):
            getattr(_L, self._free)(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class DeviceDataset(_Handle):
    _free = "aq_dataset_free"

    def __init__(self, s, h, n, d):
        self.s, self.h, self.n, self.d = s, h, n, d

    def norms(self) -> np.ndarray:
        out = np.zeros(self.n, np.float64)
        _check(_L.aq_dataset_norms(self.h, out.ctypes.data))
        return out


class DeviceCodebook(_Handle):
    _free = "aq_codebook_free"

    def __init__(self, s, h, M, k, sd):
        self.s, self.h, self.M, self.k, self.sd = s, h, M, k, sd

    def download(self) -> ProductCodebook:
        out = np.zeros(self.M * self.k * self.sd, np.float64)
        _check(_L.aq_codebook_download(self.h, out.ctypes.data))
        return ProductCodebook(self.M, self.k, self.sd, out)


class DeviceCodes(_Handle):
    _free = "aq_codes_free"

    def __init__(self, s, h, n, M, k):
        self.s, self.h, self.n, self.M, self.k = s, h, n, M, k

    @property
    def row_bytes(self) -> int:
        return int(_L.aq_codes_row_bytes(self.h))

    def download(self) -> CodeMatrix:
        out = np.zeros((self.n, self.M), np.uint32)
        _check(_L.aq_codes_download(self.h, out.ctypes.data))
        return CodeMatrix(self.n, self.M, self.k, out)

    def download_packed(self) -> np.ndarray:
        out = np.zeros((self.n, self.row_bytes), np.uint8)
        _check(_L.aq_codes_download_packed(self.h, out.ctypes.data))
        return out


# ---- weights ----------------------------------------------------------------


def _weights(w, n: int, keep: list) -> _lib.aq_weights:
    """Builds an aq_weights descriptor; `keep` holds arrays alive for the call."""
    cw = _lib.aq_weights()
    if isinstance(w, AnisotropicWeights):
        cw.mode = 0
        cw.h_parallel = w.h_parallel
        cw.h_perpendicular = w.h_perpendicular
        return cw
    if isinstance(w, ThresholdWeights):
        cw.mode = 2
        cw.threshold = w.threshold
        cw.threshold_policy = 1 if w.policy == "parallel_only" else 0
        return cw
    if isinstance(w, tuple) and len(w) == 2:
        hp = np.ascontiguousarray(w[0], np.float64)
        ho = np.ascontiguousarray(w[1], np.float64)
    else:
        seq = list(w)
        if len(seq) != n:
            raise InvalidArgument("InvalidArgument: need one AnisotropicWeights per datapoint")
        if seq and all(s == seq[0] for s in seq):
            return _weights(seq[0], n, keep)
        hp = np.array([s.h_parallel for s in seq], np.float64)
        ho = np.array([s.h_perpendicular for s in seq], np.float64)
    if hp.size != n or ho.size != n:
        raise InvalidArgument("InvalidArgument: need one AnisotropicWeights per datapoint")
    keep += [hp, ho]
    cw.mode = 1
    cw.h_parallel_arr = hp.ctypes.data
    cw.h_perpendicular_arr = ho.ctypes.data
    return cw


def _sess(session: Optional[Session]) -> Session:
    return session or Session.default()


# ---- encode (pq.hpp) ------------------------------------------------------------


def pq_quantize(data: Dataset, cb: ProductCodebook, weights, passes: int,
                threads: int = 1, session: Optional[Session] = None) -> CodeMatrix:
    """pq.hpp:581-612. `threads` is accepted for signature parity; results never
    depend on it (parallel.hpp:32-35)."""
    s = _sess(session)
    data = data if isinstance(data, Dataset) else Dataset(data)
    keep: list = []
    w = _weights(weights, data.n, keep)
    out = np.zeros((data.n, cb.M), np.uint32)
    if data.f64:  # float64 rows: the resident-dataset path
        if data.d != cb.dim():
            raise DimensionMismatch("DimensionMismatch: dataset dimension does not match codebook")
        ds, dcb, dc = s.upload_dataset(data), s.upload_codebook(cb), s.alloc_codes(data.n, cb.M, cb.k)
        _check(_L.aq_dev_pq_quantize(ds.h, dcb.h, C.byref(w), passes, dc.h))
        return dc.download()
    _check(_L.aq_pq_quantize(s.h, data.values.ctypes.data, data.n, data.d,
                             cb.dictionaries.ctypes.data, cb.M, cb.k, cb.sub_dimension,
                             C.byref(w), passes, out.ctypes.data))
    return CodeMatrix(data.n, cb.M, cb.k, out)


def pq_assign_pass(data: Dataset, cb: ProductCodebook, weights, codes: CodeMatrix,
                   sweep_to_fixed_point: bool = False, session: Optional[Session] = None):
    """detail::pq_assign_pass (pq.hpp:202-221): returns (codes, per-point losses)."""
    s = _sess(session)
    data = data if isinstance(data, Dataset) else Dataset(data)
    keep: list = []
    w = _weights(weights, data.n, keep)
    out = np.ascontiguousarray(codes.codes, np.uint32).copy()
    losses = np.zeros(data.n, np.float64)
    if data.f64:  # float64 rows: the resident-dataset path
        import torch  # device buffer for the per-point losses
        ds, dcb = s.upload_dataset(data), s.upload_codebook(cb)
        dc = s.upload_codes(CodeMatrix(data.n, cb.M, cb.k, out))
        ld = torch.zeros(max(data.n, 1), dtype=torch.float64, device=f"cuda:{s.device}")
        torch.cuda.synchronize(s.device)
        ch = C.c_uint64(0)
        _check(_L.aq_dev_pq_assign_pass(ds.h, dcb.h, C.byref(w), int(sweep_to_fixed_point),
                                        dc.h, ld.data_ptr(), C.byref(ch)))
        return dc.download(), ld[: data.n].cpu().numpy()
    _check(_L.aq_pq_assign_pass(s.h, data.values.ctypes.data, data.n, data.d,
                                cb.dictionaries.ctypes.data, cb.M, cb.k, cb.sub_dimension,
                                C.byref(w), int(sweep_to_fixed_point), out.ctypes.data,
                                losses.ctypes.data))
    return CodeMatrix(data.n, cb.M, cb.k, out), losses


def dev_pq_quantize(ds: DeviceDataset, cb: DeviceCodebook, weights, passes: int,
                    out: DeviceCodes) -> None:
    keep: list = []
    w = _weights(weights, ds.n, keep)
    _check(_L.aq_dev_pq_quantize(ds.h, cb.h, C.byref(w), passes, out.h))


def dev_pq_assign_pass(ds: DeviceDataset, cb: DeviceCodebook, weights, codes: DeviceCodes,
                       sweep_to_fixed_point: bool = False, losses_ptr: int = 0) -> int:
    keep: list = []
    w = _weights(weights, ds.n, keep)
    ch = C.c_uint64(0)
    _check(_L.aq_dev_pq_assign_pass(ds.h, cb.h, C.byref(w), int(sweep_to_fixed_point),
                                    codes.h, losses_ptr or None, C.byref(ch)))
    return ch.value


# ---- search (index.hpp) -------------------------------------------------------------


def build_lut(q, cb: ProductCodebook, session: Optional[Session] = None) -> LookupTable:
    """index.hpp:56-70 (float64 partial dot products, computed on the device)."""
    s = _sess(session)
    q = np.ascontiguousarray(q, np.float64)
    out = np.zeros(cb.M * cb.k, np.float64)
    _check(_L.aq_build_lut(s.h, q.ctypes.data, q.size, cb.dictionaries.ctypes.data, cb.M,
                           cb.k, cb.sub_dimension, out.ctypes.data))
    return LookupTable(cb.M, cb.k, out)


def adc_search(q, codes: CodeMatrix, cb: ProductCodebook, topn: int,
               session: Optional[Session] = None) -> SearchResult:
    """index.hpp:118-134: top-N by lookup-table score, (score desc, index asc)."""
    s = _sess(session)
    q = np.ascontiguousarray(q, np.float64)
    te = min(topn, codes.n) if topn >= 1 else 1
    ids = np.zeros(max(te, 1), np.uint32)
    sc = np.zeros(max(te, 1), np.float64)
    cnt = C.c_size_t(0)
    _check(_L.aq_adc_search(s.h, q.ctypes.data, q.size, codes.codes.ctypes.data, codes.n,
                            codes.M, codes.k, cb.dictionaries.ctypes.data, cb.M, cb.k,
                            cb.sub_dimension, topn, ids.ctypes.data, sc.ctypes.data,
                            C.byref(cnt)))
    return SearchResult([Hit(int(i), float(v)) for i, v in zip(ids[:cnt.value], sc[:cnt.value])])


def dev_adc_search(codes: DeviceCodes, cb: DeviceCodebook, queries, topn: int):
    """Batched adc_search over a resident index: returns (ids, scores) nq x min(topn, n)."""
    Q = np.ascontiguousarray(np.atleast_2d(queries), np.float64)
    nq = Q.shape[0]
    te = min(topn, codes.n)
    ids = np.zeros((nq, te), np.uint32)
    sc = np.zeros((nq, te), np.float64)
    _check(_L.aq_dev_adc_search(codes.h, cb.h, Q.ctypes.data, nq, topn, ids.ctypes.data,
                                sc.ctypes.data))
    return ids, sc


def dev_rerank(ds: DeviceDataset, queries, cand_ids, keep: int):
    """Exact float64 dot rerank of candidate ids (north_star A22)."""
    Q = np.ascontiguousarray(np.atleast_2d(queries), np.float64)
    cand = np.ascontiguousarray(cand_ids, np.uint32)
    nq, nc = cand.shape
    ke = min(keep, nc)
    ids = np.zeros((nq, ke), np.uint32)
    sc = np.zeros((nq, ke), np.float64)
    _check(_L.aq_dev_rerank(ds.h, Q.ctypes.data, nq, cand.ctypes.data, nc, keep,
                            ids.ctypes.data, sc.ctypes.data))
    return ids, sc


def dev_search_rerank(ds: DeviceDataset, codes: DeviceCodes, cb: DeviceCodebook, queries,
                      topn: int = 100, keep: int = 10):
    """ADC top-`topn` + exact rerank to `keep` in one device pipeline.
    Returns (adc_ids, adc_scores, ids, scores)."""
    Q = np.ascontiguousarray(np.atleast_2d(queries), np.float64)
    nq = Q.shape[0]
    te = min(topn, codes.n)
    ke = min(keep, te)
    aid = np.zeros((nq, te), np.uint32)
    asc = np.zeros((nq, te), np.float64)
    ids = np.zeros((nq, ke), np.uint32)
    sc = np.zeros((nq, ke), np.float64)
    _check(_L.aq_dev_search_rerank(ds.h, codes.h, cb.h, Q.ctypes.data, nq, topn, keep,
                                   aid.ctypes.data, asc.ctypes.data, ids.ctypes.data,
                                   sc.ctypes.data))
    return aid, asc, ids, sc


# ---- codebook update (pq.hpp:290-464) ---------------------------------------------------


def pq_codebook_update(data, codes: CodeMatrix, weights, M: int, k: int, ridge: float = -1.0,
                       session: Optional[Session] = None) -> ProductCodebook:
    """pq.hpp:356-464: joint codebook solve for fixed codes (bit-identical to the
    reference's serial normal equations + the pinned blocked Cholesky)."""
    s = _sess(session)
    data = data if isinstance(data, Dataset) else Dataset(data)
    keep: list = []
    w = _weights(weights, data.n, keep)
    out = np.zeros(k * data.d, np.float64)
    cm = np.ascontiguousarray(codes.codes, np.uint32)
    if data.f64:  # float64 rows: the resident-dataset path
        if codes.n != data.n or codes.M != M:
            raise DimensionMismatch("DimensionMismatch: code matrix does not match dataset")
        if M == 0 or data.d % M:
            raise DimensionNotDivisible("DimensionNotDivisible: dimension not divisible by M")
        ds = s.upload_dataset(data)
        dc = s.upload_codes(CodeMatrix(codes.n, M, k, cm))
        dcb = s.upload_codebook(ProductCodebook(M, k, data.d // M, out))
        _check(_L.aq_dev_pq_codebook_update(ds.h, dc.h, C.byref(w), ridge, dcb.h))
        return dcb.download()
    _check(_L.aq_pq_codebook_update(s.h, data.values.ctypes.data, data.n, data.d,
                                    cm.ctypes.data, M, k, C.byref(w), ridge, out.ctypes.data))
    return ProductCodebook(M, k, data.d // M if M else 0, out)


def assemble_selector_system(data, codes: CodeMatrix, weights, M: int, k: int,
                             session: Optional[Session] = None):
    """pq.hpp:290-343: returns (system_matrix dim x dim, rhs dim), dim = k d."""
    s = _sess(session)
    data = data if isinstance(data, Dataset) else Dataset(data)
    if codes.n != data.n or codes.M != M:
        raise DimensionMismatch("DimensionMismatch: code matrix does not match dataset")
    ds = s.upload_dataset(data)
    dc = s.upload_codes(CodeMatrix(codes.n, codes.M, k, codes.codes))
    keep: list = []
    w = _weights(weights, data.n, keep)
    dim = k * data.d
    A = np.zeros((dim, dim), np.float64)
    rhs = np.zeros(dim, np.float64)
    _check(_L.aq_dev_assemble_selector_system(ds.h, dc.h, C.byref(w), A.ctypes.data,
                                              rhs.ctypes.data))
    return A, rhs


# ---- trainers (pq.hpp:469-575) ---------------------------------------------------------


def dev_train_l2_pq(ds: DeviceDataset, M: int, k: int, config: TrainConfig = TrainConfig()):
    cfg = config.c()
    cb, cm = C.c_void_p(), C.c_void_p()
    _check(_L.aq_dev_train_l2_pq(ds.h, M, k, C.byref(cfg), C.byref(cb), C.byref(cm)))
    return (DeviceCodebook(ds.s, cb, M, k, ds.d // M), DeviceCodes(ds.s, cm, ds.n, M, k))


def dev_train_apq(ds: DeviceDataset, M: int, k: int, weights, config: TrainConfig = TrainConfig(),
                  warm_start: bool = True, loss_history: Optional[list] = None):
    cfg = config.c()
    keep: list = []
    w = _weights(weights, ds.n, keep)
    cb, cm = C.c_void_p(), C.c_void_p()
    hist = np.zeros(max(config.max_iterations, 0) + 1, np.float64)
    hl = C.c_size_t(0)
    _check(_L.aq_dev_train_apq(ds.h, M, k, C.byref(w), C.byref(cfg), int(warm_start),
                               C.byref(cb), C.byref(cm), hist.ctypes.data, C.byref(hl)))
    if loss_history is not None:
        loss_history.extend(float(v) for v in hist[: hl.value])
    return (DeviceCodebook(ds.s, cb, M, k, ds.d // M), DeviceCodes(ds.s, cm, ds.n, M, k))


@dataclass
class Codebook:  # vq.hpp:32-43: k codewords of dimension d
    k: int
    d: int
    codewords: np.ndarray  # k x d float64


@dataclass
class VqAssignment:  # vq.hpp:45-50
    assignments: np.ndarray  # n uint32
    loss_history: list


def dev_train_avq(ds: DeviceDataset, k: int, weights, config: TrainConfig = TrainConfig(),
                  loss_history: Optional[list] = None):
    """vq.hpp:243-329 on the device: (codebook as M = 1, assignments as M = 1 codes)."""
    cfg = config.c()
    keep: list = []
    w = _weights(weights, ds.n, keep)
    cb, cm = C.c_void_p(), C.c_void_p()
    hist = np.zeros(max(config.max_iterations, 0) + 1, np.float64)
    hl = C.c_size_t(0)
    _check(_L.aq_dev_train_avq(ds.h, k, C.byref(w), C.byref(cfg), C.byref(cb), C.byref(cm),
                               hist.ctypes.data, C.byref(hl)))
    if loss_history is not None:
        loss_history.extend(float(v) for v in hist[: hl.value])
    return (DeviceCodebook(ds.s, cb, 1, k, ds.d), DeviceCodes(ds.s, cm, ds.n, 1, k))


def train_avq(data, k: int, weights, config: TrainConfig = TrainConfig(),
              session: Optional[Session] = None):
    """vq.hpp:243-329: anisotropic vector quantization -> (Codebook, VqAssignment)."""
    s = _sess(session)
    ds = s.upload_dataset(data)
    hist: list = []
    cb, cm = dev_train_avq(ds, k, weights, config, hist)
    pcb, codes = cb.download(), cm.download()
    return (Codebook(k, ds.d, pcb.dictionaries.reshape(k, ds.d)),
            VqAssignment(codes.codes.reshape(-1).astype(np.uint32), hist))


def assign_point(x, cb: Codebook, w: AnisotropicWeights, session: Optional[Session] = None) -> int:
    """vq.hpp:112-132: lowest-index argmin of the anisotropic loss (M = 1 sweep)."""
    if cb.k == 0:
        raise InvalidArgument("InvalidArgument: empty codebook")
    x = np.ascontiguousarray(x, np.float64).ravel()
    if x.size != cb.d:
        raise DimensionMismatch("DimensionMismatch: datapoint dimension does not match codebook")
    return int(pq_assign_point(x, np.zeros(1, np.uint32),
                               ProductCodebook(1, cb.k, cb.d, cb.codewords), w,
                               session=session)[0])


def update_codeword(d: int, points, weights, ridge: float = -1.0,
                    session: Optional[Session] = None) -> np.ndarray:
    """vq.hpp:139-192: closed-form codeword of weighted points (the device M = 1
    update with every point in partition 0)."""
    pts = np.ascontiguousarray(points, np.float64).ravel()
    if d == 0 or pts.size == 0 or pts.size % d:
        raise InvalidArgument("InvalidArgument: points must be a non-empty multiple of d")
    m = pts.size // d
    ws = weights if isinstance(weights, (list, tuple)) else None
    if ws is not None and len(ws) != m:
        raise InvalidArgument("InvalidArgument: need one weight per point")
    out = pq_codebook_update(pts.reshape(m, d), CodeMatrix(m, 1, 1, np.zeros((m, 1), np.uint32)),
                             weights, 1, 1, ridge, session=session)
    return out.dictionaries.copy()


def vq_quantize(data, cb: Codebook, weights, threads: int = 1,
                session: Optional[Session] = None) -> np.ndarray:
    """vq.hpp:332-343: one assignment pass against a fixed VQ codebook."""
    data = data if isinstance(data, Dataset) else Dataset(data)
    if data.d != cb.d:
        raise DimensionMismatch("DimensionMismatch: dataset dimension does not match codebook")
    if data.n == 0:
        return np.zeros(0, np.uint32)
    codes, _ = pq_assign_pass(data, ProductCodebook(1, cb.k, cb.d, cb.codewords), weights,
                              CodeMatrix(data.n, 1, cb.k, np.zeros((data.n, 1), np.uint32)),
                              session=session)
    return codes.codes.reshape(-1).copy()


def train_l2_pq(data, M: int, k: int, config: TrainConfig = TrainConfig(),
                session: Optional[Session] = None):
    """pq.hpp:469-501: classical PQ (independent k-means per subspace, seed + m)."""
    s = _sess(session)
    ds = s.upload_dataset(data)
    cb, cm = dev_train_l2_pq(ds, M, k, config)
    return cb.download(), cm.download()


def train_apq(data, M: int, k: int, weights, config: TrainConfig = TrainConfig(),
              warm_start: bool = True, loss_history: Optional[list] = None,
              session: Optional[Session] = None):
    """pq.hpp:513-575: alternating anisotropic PQ trainer."""
    s = _sess(session)
    ds = s.upload_dataset(data)
    cb, cm = dev_train_apq(ds, M, k, weights, config, warm_start, loss_history)
    return cb.download(), cm.download()


# ---- multi-device session (csrc/multi.cu) ---------------------------------------------


class MultiSession:
    """Row shards over the GPUs of one box from one process (one session per
    entry of `devices`; a device may carry several shards). pq_quantize and
    adc_search equal the single-device calls; train_apq equals them for one
    shard and re-associates the float64 partial sums at shard boundaries for
    more (include/anisoq_b200.h)."""

    def __init__(self, devices):
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(_L.aq_multi_create(devs, len(devices), C.byref(h)))
        self.h = h
        self.devices = list(devices)

    @property
    def shards(self) -> int:
        return _L.aq_multi_shards(self.h)

    def close(self) -> None:
        if self.h:
            _L.aq_multi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def pq_quantize(self, data, cb: ProductCodebook, weights, passes: int) -> CodeMatrix:
        data = data if isinstance(data, Dataset) else Dataset(data)
        if data.f64:
            raise Unsupported("Unsupported: multi-device calls take float32-exact rows")
        keep: list = []
        w = _weights(weights, data.n, keep)
        out = np.zeros((data.n, cb.M), np.uint32)
        _check(_L.aq_multi_pq_quantize(self.h, data.values.ctypes.data, data.n, data.d,
                                       cb.dictionaries.ctypes.data, cb.M, cb.k,
                                       cb.sub_dimension, C.byref(w), passes, out.ctypes.data))
        return CodeMatrix(data.n, cb.M, cb.k, out)

    def adc_search(self, queries, codes: CodeMatrix, cb: ProductCodebook, topn: int):
        Q = np.ascontiguousarray(np.atleast_2d(queries), np.float64)
        cm = np.ascontiguousarray(codes.codes, np.uint32)
        te = min(topn, codes.n) if topn >= 1 else 1
        ids = np.zeros((len(Q), te), np.uint32)
        sc = np.zeros((len(Q), te), np.float64)
        _check(_L.aq_multi_adc_search(self.h, Q.ctypes.data, len(Q), Q.shape[1], cm.ctypes.data,
                                      codes.n, codes.M, codes.k, cb.dictionaries.ctypes.data,
                                      cb.M, cb.k, cb.sub_dimension, topn, ids.ctypes.data,
                                      sc.ctypes.data))
        return ids, sc

    def train_apq(self, data, M: int, k: int, weights, config: TrainConfig = TrainConfig(),
                  warm_start: bool = True, loss_history: Optional[list] = None):
        data = data if isinstance(data, Dataset) else Dataset(data)
        if data.f64:
            raise Unsupported("Unsupported: multi-device calls take float32-exact rows")
        keep: list = []
        w = _weights(weights, data.n, keep)
        cfg = config.c()
        dic = np.zeros(k * data.d, np.float64)
        codes = np.zeros((data.n, M), np.uint32)
        hist = np.zeros(max(config.max_iterations, 0) + 1, np.float64)
        hl = C.c_size_t(0)
        _check(_L.aq_multi_train_apq(self.h, data.values.ctypes.data, data.n, data.d, M, k,
                                     C.byref(w), C.byref(cfg), int(warm_start), dic.ctypes.data,
                                     codes.ctypes.data, hist.ctypes.data, C.byref(hl)))
        if loss_history is not None:
            loss_history.extend(float(v) for v in hist[: hl.value])
        return ProductCodebook(M, k, data.d // M, dic), CodeMatrix(data.n, M, k, codes)


# ---- single-point API, exact search, evaluation (pq.hpp:256, index.hpp:137-332) ---------


def pq_assign_point(x, current_codes, cb: ProductCodebook, w: AnisotropicWeights,
                    sweep_order=None, session: Optional[Session] = None) -> np.ndarray:
    """pq.hpp:256-282: one coordinate-descent pass for a single float64 point
    over `sweep_order` (default 0..M-1; subspaces may repeat)."""
    s = _sess(session)
    x = np.ascontiguousarray(x, np.float64)
    cur = np.ascontiguousarray(current_codes, np.uint32)
    if x.size != cb.dim():
        raise DimensionMismatch("DimensionMismatch: datapoint dimension does not match codebook")
    if cur.size != cb.M:
        raise DimensionMismatch("DimensionMismatch: need one current code per subspace")
    order = np.ascontiguousarray([] if sweep_order is None else sweep_order, np.uint64)
    out = np.zeros(cb.M, np.uint32)
    _check(_L.aq_pq_assign_point_order(s.h, x.ctypes.data, x.size, cur.ctypes.data,
                                       cb.dictionaries.ctypes.data, cb.M, cb.k,
                                       cb.sub_dimension, w.h_parallel, w.h_perpendicular,
                                       order.ctypes.data if order.size else None, order.size,
                                       out.ctypes.data))
    return out


def dev_exact_search(ds: DeviceDataset, queries, depth: int):
    """exact_ground_truth (index.hpp:150-162): exact float64 MIPS top-`depth`."""
    Q = np.ascontiguousarray(np.atleast_2d(queries), np.float64)
    nq = Q.shape[0]
    te = min(depth, ds.n)
    ids = np.zeros((nq, te), np.uint32)
    sc = np.zeros((nq, te), np.float64)
    _check(_L.aq_dev_exact_search(ds.h, Q.ctypes.data, nq, depth, ids.ctypes.data,
                                  sc.ctypes.data))
    return ids, sc


def exact_search(q, data, topn: int, session: Optional[Session] = None) -> SearchResult:
    """index.hpp:137-147."""
    s = _sess(session)
    data = data if isinstance(data, Dataset) else Dataset(data)
    if data.n == 0:
        raise EmptyDataset("EmptyDataset: empty dataset")
    if topn < 1:
        raise InvalidArgument("InvalidArgument: topn must be >= 1")
    q = np.ascontiguousarray(q, np.float64)
    if q.size != data.d:
        raise DimensionMismatch("DimensionMismatch: query dimension does not match dataset")
    ids, sc = dev_exact_search(s.upload_dataset(data), q[None, :], topn)
    return SearchResult([Hit(int(i), float(v)) for i, v in zip(ids[0], sc[0])])


def _seq_dot(a: np.ndarray, b: np.ndarray) -> float:
    """detail::dot order (geometry.hpp:170-174): products rounded, summed in order."""
    p = np.asarray(a, np.float64) * np.asarray(b, np.float64)
    return float(np.add.accumulate(p)[-1]) if p.size else 0.0


@dataclass
class EvalOptions:
    recall_ns: tuple = (1, 10, 100)
    kk: int = 10
    threads: int = 1
    ground_truth: Optional[np.ndarray] = None
    # extension: search and time the queries one at a time against the
    # device-resident index (the reference's per-query latency,
    # index.hpp:254-259); default: one batch, latency = batch time / queries
    per_query_latency: bool = False


@dataclass
class LatencySummary:  # index.hpp:164-168
    mean_us: float = 0.0
    p50_us: float = 0.0
    p99_us: float = 0.0


@dataclass
class EvalReport:
    num_queries: int
    num_datapoints: int
    recall_1_at_n: dict
    kk: int
    recall_k_at_k: float
    relative_error_mean: float
    relative_error_p50: float
    relative_error_p90: float
    relative_error_p99: float
    relative_error_max: float
    latency: LatencySummary = field(default_factory=LatencySummary)

    def write_text(self) -> str:
        """EvalReport::write_text (index.hpp:183-197): one `name value` per
        line, values in the default iostream format (%g)."""
        out = [f"num_queries {self.num_queries}", f"num_datapoints {self.num_datapoints}"]
        out += [f"recall_1@{n} {r:g}" for n, r in sorted(self.recall_1_at_n.items())]
        out += [f"recall_{self.kk}@{self.kk} {self.recall_k_at_k:g}",
                f"relative_error_top1_mean {self.relative_error_mean:g}",
                f"relative_error_top1_p50 {self.relative_error_p50:g}",
                f"relative_error_top1_p90 {self.relative_error_p90:g}",
                f"relative_error_top1_p99 {self.relative_error_p99:g}",
                f"relative_error_top1_max {self.relative_error_max:g}",
                f"latency_mean_us {self.latency.mean_us:g}",
                f"latency_p50_us {self.latency.p50_us:g}",
                f"latency_p99_us {self.latency.p99_us:g}"]
        return "\n".join(out) + "\n"


def evaluate(queries, data, codes: CodeMatrix, cb: ProductCodebook,
             options: EvalOptions = EvalOptions(), session: Optional[Session] = None) -> EvalReport:
    """index.hpp:213-332 with the searches on the device (batched adc_search and
    exact ground truth); the recall / relative-error bookkeeping follows the
    reference line by line. Latency: batch time / queries, or each query's own
    search time with options.per_query_latency."""
    s = _sess(session)
    Q = np.ascontiguousarray(np.atleast_2d(queries), np.float64)
    data = data if isinstance(data, Dataset) else Dataset(data)
    if Q.shape[0] == 0:
        raise EmptyDataset("EmptyDataset: no queries")
    if data.n == 0:
        raise EmptyDataset("EmptyDataset: empty dataset")
    if codes.n != data.n:
        raise DimensionMismatch("DimensionMismatch: code matrix does not match dataset")
    if Q.shape[1] != data.d or data.d != cb.dim():
        raise DimensionMismatch("DimensionMismatch: query/dataset/codebook dimensions differ")
    if not options.recall_ns:
        raise InvalidArgument("InvalidArgument: need at least one N")
    depth = min(max([options.kk, *options.recall_ns]), data.n)
    ds = s.upload_dataset(data)
    if options.ground_truth is not None:
        gt = np.asarray(options.ground_truth)
        if gt.shape[0] != Q.shape[0]:
            raise GroundTruthMismatch(f"GroundTruthMismatch: ground truth has {gt.shape[0]} rows, "
                                      f"need {Q.shape[0]}")
        if gt.ndim < 2 or gt.shape[1] < depth:
            raise GroundTruthMismatch(f"GroundTruthMismatch: ground truth rows need at least "
                                      f"{depth} entries")
    else:
        gt, _ = dev_exact_search(ds, Q, depth)
    dc = s.upload_codes(codes)
    dcb = s.upload_codebook(cb)
    nq = Q.shape[0]
    dev_adc_search(dc, dcb, Q[:1], depth)  # warm-up outside the timed region
    if options.per_query_latency:
        rows, lat = [], []
        for qi in range(nq):
            t0 = time.perf_counter()
            r_ids, _ = dev_adc_search(dc, dcb, Q[qi:qi + 1], depth)
            lat.append((time.perf_counter() - t0) * 1e6)
            rows.append(r_ids[0])
        ids = np.stack(rows)
    else:
        t0 = time.perf_counter()
        ids, _ = dev_adc_search(dc, dcb, Q, depth)
        lat = [(time.perf_counter() - t0) * 1e6 / nq] * nq
    lat = sorted(lat)  # index.hpp:322-330
    latency = LatencySummary(float(np.add.accumulate(lat)[-1] / nq),
                             lat[min(nq - 1, int(0.50 * nq))], lat[min(nq - 1, int(0.99 * nq))])
    kk = min(options.kk, data.n)
    found = {n_: 0 for n_ in options.recall_ns}
    overlap = np.zeros(nq)
    rel = np.zeros(nq)
    for qi in range(nq):
        top1 = int(gt[qi][0])
        for n_ in options.recall_ns:
            if top1 in ids[qi][: min(n_, ids.shape[1])].tolist():
                found[n_] += 1
        overlap[qi] = len(set(ids[qi][:kk].tolist()) & set(int(v) for v in gt[qi][:kk])) / kk
        exact = _seq_dot(Q[qi], data.values[top1])
        rec = np.concatenate([cb.codeword(m, int(c)) for m, c in enumerate(codes.codes[top1])])
        approx = _seq_dot(Q[qi], rec)
        rel[qi] = abs((exact - approx) / exact) if exact != 0.0 else abs(exact - approx)
    srt = np.sort(rel)

    def quantile(p):
        idx = int(math.ceil(p * len(srt)))
        return float(srt[min(len(srt) - 1, 0 if idx == 0 else idx - 1)])

    return EvalReport(nq, data.n, {n_: found[n_] / nq for n_ in options.recall_ns}, kk,
                      float(np.add.accumulate(overlap)[-1] / nq),
                      float(np.add.accumulate(srt)[-1] / nq), quantile(0.5), quantile(0.9),
                      quantile(0.99), float(srt[-1]), latency)


# ---- on-disk formats (pq.hpp:614-730, dataset.hpp:122-219) -------------------------------
# Host I/O, byte-compatible with the reference's files.

import struct as _struct


def save_codebook(cb: ProductCodebook, path: str) -> None:
    """AQCB container: magic, version 1, M, k, d (LE uint32), float32 dictionaries."""
    with open(path, "wb") as f:
        f.write(b"AQCB" + _struct.pack("<4I", 1, cb.M, cb.k, cb.dim()))
        f.write(np.asarray(cb.dictionaries, np.float64).astype("<f4").tobytes())


def load_codebook(path: str) -> ProductCodebook:
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise MalformedFile(f"MalformedFile: cannot open {path}")
    if len(raw) < 4 or raw[:4] != b"AQCB":
        raise MalformedFile(f"MalformedFile: {path}: bad magic")
    if len(raw) < 20:
        raise MalformedFile(f"MalformedFile: {path}: truncated header")
    version, M, k, d = _struct.unpack("<4I", raw[4:20])
    if version != 1:
        raise MalformedFile(f"MalformedFile: {path}: unsupported version {version}")
    if M == 0 or d == 0 or d % M:
        raise MalformedFile(f"MalformedFile: {path}: inconsistent shape")
    cnt = k * d
    if len(raw) < 20 + 4 * cnt:
        raise MalformedFile(f"MalformedFile: {path}: truncated dictionaries")
    vals = np.frombuffer(raw, "<f4", cnt, 20).astype(np.float64)
    return ProductCodebook(M, k, d // M, vals)


def save_codes(cm: CodeMatrix, path: str) -> None:
    """n, M, k (LE uint32) then codes row-major as uint8 (k <= 256) or uint16."""
    if cm.k > 65536:
        raise InvalidArgument("InvalidArgument: code serialization supports k <= 65536")
    dt = "<u1" if cm.k <= 256 else "<u2"
    with open(path, "wb") as f:
        f.write(_struct.pack("<3I", cm.n, cm.M, cm.k))
        f.write(np.asarray(cm.codes).astype(dt).tobytes())


def load_codes(path: str) -> CodeMatrix:
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise MalformedFile(f"MalformedFile: cannot open {path}")
    if len(raw) < 12:
        raise MalformedFile(f"MalformedFile: {path}: truncated header")
    n, M, k = _struct.unpack("<3I", raw[:12])
    if M == 0:
        raise MalformedFile(f"MalformedFile: {path}: M must be positive")
    dt = "<u1" if k <= 256 else "<u2"
    need = n * M * (1 if k <= 256 else 2)
    if len(raw) < 12 + need:
        raise MalformedFile(f"MalformedFile: {path}: truncated codes")
    codes = np.frombuffer(raw, dt, n * M, 12).astype(np.uint32)
    if codes.size and codes.max() >= k:
        raise CodeOutOfRange(f"CodeOutOfRange: {path}: stored code exceeds k")
    return CodeMatrix(n, M, k, codes.reshape(n, M))


def read_fvecs(path: str) -> Dataset:
    """fvecs: per record an LE int32 dimension then that many float32 values."""
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise MalformedFile(f"MalformedFile: cannot open {path}")
    if not raw:
        return Dataset(np.zeros((0, 1), np.float32))
    if len(raw) < 4:
        raise MalformedFile(f"MalformedFile: {path}: truncated record header")
    d = _struct.unpack("<i", raw[:4])[0]
    if d <= 0:
        raise MalformedFile(f"MalformedFile: {path}: non-positive dimension")
    rec = 4 + 4 * d
    if len(raw) % rec:
        raise MalformedFile(f"MalformedFile: {path}: truncated record {len(raw) // rec}")
    arr = np.frombuffer(raw, np.uint8).reshape(-1, rec)
    dims = arr[:, :4].copy().view("<i4").ravel()
    if (dims != d).any():
        bad = int(np.argmax(dims != d))
        raise MalformedFile(f"MalformedFile: {path}: inconsistent dimension at record {bad}")
    vals = arr[:, 4:].copy().view("<f4").reshape(-1, d)
    if not np.isfinite(vals).all():
        bad = int(np.argmax(~np.isfinite(vals).all(axis=1)))
        raise MalformedFile(f"MalformedFile: {path}: non-finite value in record {bad}")
    if (np.einsum("ij,ij->i", vals.astype(np.float64), vals.astype(np.float64)) == 0).any():
        bad = int(np.argmax(~vals.any(axis=1)))
        raise ZeroNormDatapoint(f"ZeroNormDatapoint: {path}: row {bad} has zero norm")
    return Dataset(vals.astype(np.float32))


def write_fvecs(ds: Dataset, path: str) -> None:
    ds = ds if isinstance(ds, Dataset) else Dataset(ds)
    n, d = ds.values.shape
    out = np.empty((n, 1 + d), "<f4")
    out[:, 0] = np.frombuffer(_struct.pack("<i", d), "<f4")[0]
    out[:, 1:] = ds.values
    with open(path, "wb") as f:
        f.write(out.tobytes())


def read_ivecs(path: str) -> list:
    raw = open(path, "rb").read()
    out, pos = [], 0
    while pos < len(raw):
        if pos + 4 > len(raw):
            raise MalformedFile(f"MalformedFile: {path}: truncated header")
        c = _struct.unpack("<i", raw[pos:pos + 4])[0]
        pos += 4
        if c < 0:
            raise MalformedFile(f"MalformedFile: {path}: negative count")
        if pos + 4 * c > len(raw):
            raise MalformedFile(f"MalformedFile: {path}: truncated record {len(out)}")
        out.append(np.frombuffer(raw, "<i4", c, pos).copy())
        pos += 4 * c
    return out


def write_ivecs(rows, path: str) -> None:
    with open(path, "wb") as f:
        for r in rows:
            r = np.asarray(r, "<i4")
            f.write(_struct.pack("<i", r.size) + r.tobytes())


# ---- host generator and dataset helpers (rng.hpp:28-89, dataset.hpp:225-290) -------------


class Rng:
    """The reference generator contract (rng.hpp): splitmix64, 53-bit uniform
    doubles, unbiased next_below, Box-Muller normals with one cached spare,
    sample_distinct = first k of a partial Fisher-Yates shuffle of [0, n)."""

    _M = (1 << 64) - 1

    def __init__(self, seed: int):
        self._s = seed & self._M
        self._spare = None

    def next_u64(self) -> int:
        self._s = (self._s + 0x9E3779B97F4A7C15) & self._M
        z = self._s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self._M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self._M
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def next_below(self, n: int) -> int:
        reject_below = ((1 << 64) - n) % n
        while True:
            r = self.next_u64()
            if r >= reject_below:
                return r % n

    def next_gaussian(self) -> float:
        if self._spare is not None:
            v, self._spare = self._spare, None
            return v
        u1 = self.next_double()
        while u1 <= 0.0:
            u1 = self.next_double()
        u2 = self.next_double()
        radius = math.sqrt(-2.0 * math.log(u1))
        angle = 6.283185307179586476925286766559 * u2
        self._spare = radius * math.sin(angle)
        return radius * math.cos(angle)

    def sample_distinct(self, n: int, k: int) -> list:
        moved: dict = {}
        out = []
        for i in range(min(k, n)):
            j = i + self.next_below(n - i)
            vi, vj = moved.get(i, i), moved.get(j, j)
            moved[i], moved[j] = vj, vi
            out.append(vj)
        return out


def generate_synthetic(kind: str, n: int, d: int, seed: int, centers: int = 16,
                       spread: float = 0.25, normalize: bool = False) -> Dataset:
    """dataset.hpp:245-290: 'uniform_sphere' or 'gaussian_mixture', one Rng
    stream, values rounded to float32 (device-exact). Pure host code (slow for
    large n; the bench uses workload.py's vectorised generators)."""
    if n < 1 or d < 2:
        raise InvalidArgument("InvalidArgument: need n >= 1 and d >= 2")
    r = Rng(seed)
    v = np.empty((n, d), np.float64)

    def unit_row():
        while True:
            row = [r.next_gaussian() for _ in range(d)]
            ss = 0.0
            for t in row:
                ss += t * t
            if ss != 0.0:
                inv = 1.0 / math.sqrt(ss)
                return [t * inv for t in row]

    if kind == "uniform_sphere":
        for i in range(n):
            v[i] = unit_row()
        normalized = True
    elif kind == "gaussian_mixture":
        if centers < 1:
            raise InvalidArgument("InvalidArgument: need at least one center")
        ctr = [unit_row() for _ in range(centers)]
        for i in range(n):
            c = ctr[r.next_below(centers)]
            row = [c[j] + spread * r.next_gaussian() for j in range(d)]
            if normalize:
                ss = 0.0
                for t in row:
                    ss += t * t
                if ss == 0.0:
                    raise ZeroNormDatapoint("ZeroNormDatapoint: degenerate mixture sample")
                inv = 1.0 / math.sqrt(ss)
                row = [t * inv for t in row]
            v[i] = row
        normalized = normalize
    else:
        raise InvalidArgument(f"InvalidArgument: unknown kind {kind!r}")
    ds = Dataset(v.astype(np.float32).astype(np.float64))
    ds.normalized = normalized
    return ds


def unit_normalize(ds: Dataset) -> np.ndarray:
    """dataset.hpp:225-236: rows scaled to unit norm (float64; generally not
    float32-exact, so devices hold the result as float64 rows)."""
    x = np.asarray(ds.values if isinstance(ds, Dataset) else ds, np.float64)
    norms = np.sqrt(np.add.accumulate(x * x, axis=1)[:, -1])  # dataset.hpp:55-59 order
    if np.any(norms == 0.0):
        i = int(np.nonzero(norms == 0.0)[0][0])
        raise ZeroNormDatapoint(f"ZeroNormDatapoint: row {i} has zero norm")
    return x / norms[:, None]
