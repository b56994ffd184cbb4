"""ctypes loader for the CPU oracle (``liboracle.so``, built from ld_oracle.c).

TEST INFRASTRUCTURE ONLY: may be imported by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.  The product package ``paper_2212_09460_b200`` never
imports it.  Every wrapper is argument marshalling around the C functions
documented (with their paper citations) in ``ld_oracle.h``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ld_oracle.c")
HDR = os.path.join(HERE, "ld_oracle.h")
LIB = os.path.join(HERE, "liboracle.so")

SENTINEL = (-1, -1, 0)


class Peak(ctypes.Structure):
    _fields_ = [("theta_bin", ctypes.c_int32), ("rho_bin", ctypes.c_int32),
                ("votes", ctypes.c_uint32)]


PEAK_DTYPE = np.dtype([("theta_bin", "<i4"), ("rho_bin", "<i4"), ("votes", "<u4")])


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain ``gcc -O2`` (no SIMD intrinsics, no OpenMP)."""
    stale = (not os.path.exists(LIB) or
             max(os.path.getmtime(SRC), os.path.getmtime(HDR)) > os.path.getmtime(LIB))
    if force or stale:
        tmp = LIB + ".tmp%d" % os.getpid()
        # -ffp-contract=off: every double product and quotient of the lanes
        # module (R27, R28) is rounded on its own, as the header states
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-Wextra", "-Werror",
                               "-ffp-contract=off", "-fPIC", "-shared", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        i32, i64, u32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        L.ldo_rho_offset.argtypes = [i32, i32]
        L.ldo_rho_offset.restype = i32
        L.ldo_sobel_magnitude.argtypes = [P, i32, i32, i64, P]
        L.ldo_sobel_binarize.argtypes = [P, i32, i32, i64, i32, P]
        L.ldo_sobel_magnitude_ex.argtypes = [P, i32, i32, i64, i32, P]
        L.ldo_sobel_binarize_ex.argtypes = [P, i32, i32, i64, i32, i32, P]
        L.ldo_compact.argtypes = [P, i32, i32, P, i64, P]
        L.ldo_hough_accumulate.argtypes = [P, i64, i32, i32, i32, P, P, P]
        L.ldo_hough_peaks.argtypes = [P, i32, i32, i32, i32, u32, i32, P, P]
        L.ldo_hough_accumulate_f64.argtypes = [P, i64, i32, i32, i32, P, P, P]
        L.ldo_hough_peaks_nms.argtypes = [P, i32, i32, i32, i32, u32, u32, u32, i32, P, P]
        L.ldo_peak_to_line.argtypes = [Peak, i32, i32, i32, P, P, P, P]
        L.ldo_extract_segments.argtypes = [P, i32, i32, i64, Peak, i32, P, P, i32, i32, P, i32,
                                           P]
        L.ldo_detect.argtypes = [P, i32, i32, i64, i32, i32, P, P, i32, i32, u32, i32,
                                 P, P, P, P, P, P]
        for f in ("ldo_sobel_magnitude", "ldo_sobel_binarize", "ldo_sobel_magnitude_ex",
                  "ldo_sobel_binarize_ex", "ldo_compact",
                  "ldo_hough_accumulate", "ldo_hough_peaks", "ldo_detect"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise OracleError("%s failed with code %d" % (what, rc))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _gray(gray: np.ndarray):
    g = np.ascontiguousarray(gray, dtype=np.uint8)
    assert g.ndim == 2
    return g


def rho_offset(width: int, height: int) -> int:
    return int(lib().ldo_rho_offset(width, height))


def sobel_magnitude(gray: np.ndarray) -> np.ndarray:
    g = _gray(gray)
    h, w = g.shape
    mag = np.empty((h, w), np.int32)
    _check(lib().ldo_sobel_magnitude(_ptr(g), w, h, w, _ptr(mag)), "sobel_magnitude")
    return mag


def sobel_binarize(gray: np.ndarray, threshold: int) -> np.ndarray:
    g = _gray(gray)
    h, w = g.shape
    out = np.empty((h, w), np.uint8)
    _check(lib().ldo_sobel_binarize(_ptr(g), w, h, w, int(threshold), _ptr(out)),
           "sobel_binarize")
    return out


ZERO_PAD, CLAMP_255 = 1, 2  # ldo_sobel_*_ex flags (NEXT 4)


def sobel_magnitude_ex(gray: np.ndarray, flags: int) -> np.ndarray:
    g = _gray(gray)
    h, w = g.shape
    mag = np.empty((h, w), np.int32)
    _check(lib().ldo_sobel_magnitude_ex(_ptr(g), w, h, w, int(flags), _ptr(mag)),
           "sobel_magnitude_ex")
    return mag


def sobel_binarize_ex(gray: np.ndarray, threshold: int, flags: int) -> np.ndarray:
    g = _gray(gray)
    h, w = g.shape
    out = np.empty((h, w), np.uint8)
    _check(lib().ldo_sobel_binarize_ex(_ptr(g), w, h, w, int(threshold), int(flags), _ptr(out)),
           "sobel_binarize_ex")
    return out


def compact(binary: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(binary, dtype=np.uint8)
    h, w = b.shape
    edges = np.empty(max(h * w, 1), np.uint32)
    n = ctypes.c_int64(0)
    _check(lib().ldo_compact(_ptr(b), w, h, _ptr(edges), h * w, ctypes.byref(n)), "compact")
    return edges[: n.value].copy()


def hough_accumulate(edges: np.ndarray, width: int, height: int, cos_q15: np.ndarray,
                     sin_q15: np.ndarray) -> np.ndarray:
    e = np.ascontiguousarray(edges, dtype=np.uint32)
    c = np.ascontiguousarray(cos_q15, dtype=np.int32)
    s = np.ascontiguousarray(sin_q15, dtype=np.int32)
    n_theta = c.shape[0]
    assert s.shape[0] == n_theta
    n_rho = 2 * rho_offset(width, height) + 1
    acc = np.empty((n_theta, n_rho), np.uint32)
    _check(lib().ldo_hough_accumulate(_ptr(e), e.shape[0], width, height, n_theta,
                                      _ptr(c), _ptr(s), _ptr(acc)), "hough_accumulate")
    return acc


def hough_peaks(acc: np.ndarray, half_theta: int, half_rho: int, min_votes: int,
                k: int) -> tuple[np.ndarray, int]:
    a = np.ascontiguousarray(acc, dtype=np.uint32)
    n_theta, n_rho = a.shape
    peaks = np.empty(k, PEAK_DTYPE)
    n = ctypes.c_int32(0)
    _check(lib().ldo_hough_peaks(_ptr(a), n_theta, n_rho, half_theta, half_rho,
                                 int(min_votes), k, _ptr(peaks), ctypes.byref(n)),
           "hough_peaks")
    return peaks, int(n.value)


def detect(gray: np.ndarray, threshold: int, cos_q15: np.ndarray, sin_q15: np.ndarray,
           half_theta: int, half_rho: int, min_votes: int, k: int,
           want_binary: bool = True, want_acc: bool = True) -> dict:
    """One frame through the whole oracle pipeline; returns every intermediate."""
    g = _gray(gray)
    h, w = g.shape
    c = np.ascontiguousarray(cos_q15, dtype=np.int32)
    s = np.ascontiguousarray(sin_q15, dtype=np.int32)
    n_theta = c.shape[0]
    n_rho = 2 * rho_offset(w, h) + 1
    binary = np.empty((h, w), np.uint8) if want_binary else None
    edges = np.empty(h * w, np.uint32)
    acc = np.empty((n_theta, n_rho), np.uint32) if want_acc else None
    peaks = np.empty(k, PEAK_DTYPE)
    ne = ctypes.c_int64(0)
    npk = ctypes.c_int32(0)
    nul = ctypes.c_void_p(None)
    _check(lib().ldo_detect(_ptr(g), w, h, w, int(threshold), n_theta, _ptr(c), _ptr(s),
                            half_theta, half_rho, int(min_votes), k,
                            _ptr(binary) if binary is not None else nul, _ptr(edges),
                            ctypes.byref(ne), _ptr(acc) if acc is not None else nul,
                            _ptr(peaks), ctypes.byref(npk)), "detect")
    return {"binary": binary, "edges": edges[: ne.value].copy(), "n_edges": int(ne.value),
            "acc": acc, "peaks": peaks, "n_peaks": int(npk.value)}


# ----------------------------------------------------------------------------
# NEXT 3: lanes module (ld_oracle.h R26-R28)
# ----------------------------------------------------------------------------
SEG_DTYPE = np.dtype([("x0", "<i4"), ("y0", "<i4"), ("x1", "<i4"), ("y1", "<i4")])


def hough_peaks_nms(acc: np.ndarray, half_theta: int, half_rho: int, min_votes: int,
                    ratio_num: int, ratio_den: int, k: int) -> tuple[np.ndarray, int]:
    a = np.ascontiguousarray(acc, dtype=np.uint32)
    n_theta, n_rho = a.shape
    peaks = np.empty(k, PEAK_DTYPE)
    n = ctypes.c_int32(0)
    _check(lib().ldo_hough_peaks_nms(_ptr(a), n_theta, n_rho, half_theta, half_rho,
                                     int(min_votes), int(ratio_num), int(ratio_den), k,
                                     _ptr(peaks), ctypes.byref(n)), "hough_peaks_nms")
    return peaks, int(n.value)


def _peak(p) -> Peak:
    return Peak(int(p[0]), int(p[1]), int(p[2]))


def peak_to_line(peak, width: int, height: int, cos_q15: np.ndarray,
                 sin_q15: np.ndarray):
    """peak = (theta_bin, rho_bin, votes).  Returns (x0, y0, x1, y1) or None."""
    c = np.ascontiguousarray(cos_q15, dtype=np.int32)
    s = np.ascontiguousarray(sin_q15, dtype=np.int32)
    seg = np.zeros(1, SEG_DTYPE)
    hit = ctypes.c_int32(0)
    _check(lib().ldo_peak_to_line(_peak(peak), width, height, c.shape[0], _ptr(c), _ptr(s),
                                  _ptr(seg), ctypes.byref(hit)), "peak_to_line")
    return tuple(int(v) for v in seg[0]) if hit.value else None


def extract_segments(binary: np.ndarray, peak, cos_q15: np.ndarray, sin_q15: np.ndarray,
                     fill_gap: int = 20, min_len: int = 40, cap: int = 1024):
    """Returns the list of (x0, y0, x1, y1) segments in walk order."""
    b = np.ascontiguousarray(binary, dtype=np.uint8)
    h, w = b.shape
    c = np.ascontiguousarray(cos_q15, dtype=np.int32)
    s = np.ascontiguousarray(sin_q15, dtype=np.int32)
    segs = np.zeros(max(cap, 1), SEG_DTYPE)
    n = ctypes.c_int32(0)
    _check(lib().ldo_extract_segments(_ptr(b), w, h, w, _peak(peak), c.shape[0], _ptr(c),
                                      _ptr(s), fill_gap, min_len, _ptr(segs), cap,
                                      ctypes.byref(n)), "extract_segments")
    return [tuple(int(v) for v in segs[i]) for i in range(min(n.value, cap))], int(n.value)


def hough_accumulate_f64(edges: np.ndarray, width: int, height: int, cos_f64: np.ndarray,
                         sin_f64: np.ndarray) -> np.ndarray:
    """SPEC float64 trig mode (ld_oracle.h, DESIGN R29)."""
    e = np.ascontiguousarray(edges, dtype=np.uint32)
    c = np.ascontiguousarray(cos_f64, dtype=np.float64)
    s = np.ascontiguousarray(sin_f64, dtype=np.float64)
    n_theta = c.shape[0]
    n_rho = 2 * rho_offset(width, height) + 1
    acc = np.empty((n_theta, n_rho), np.uint32)
    _check(lib().ldo_hough_accumulate_f64(_ptr(e) if e.size else None, e.size, width, height,
                                          n_theta, _ptr(c), _ptr(s), _ptr(acc)),
           "hough_accumulate_f64")
    return acc


# ----------------------------------------------------------------------------
# Frame-parallel harness (test/baseline infrastructure, no arithmetic of its
# own): independent frames go to a thread pool.  ctypes releases the GIL for
# the duration of each C call, so N threads run N single-threaded oracle
# frames at once -- SURVEY 8(d) "frame-parallel across all cores".
# ----------------------------------------------------------------------------
def host_cores() -> int:
    """Cores this process may run on (the affinity mask, else os.cpu_count())."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover - non-Linux
        return os.cpu_count() or 1


def cpu_model() -> str:
    """The host CPU model string (/proc/cpuinfo), for the bench record."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def map_frames(fn, items, workers: int | None = None):
    """[fn(item) for item in items] on a pool of `workers` threads (default:
    every host core), results in input order.  fn should spend its time in
    oracle C calls (which run without the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    lib()  # load once, before the threads
    items = list(items)
    workers = max(1, min(workers or host_cores(), len(items) or 1))
    if workers == 1:
        return [fn(it) for it in items]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(fn, items))
