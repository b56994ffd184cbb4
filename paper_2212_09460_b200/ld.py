"""Thin Python binding of libld.so (include/ld.h): argument marshalling only.

Two layers:
  * ``ld_*`` -- the C ABI one-to-one (same names, same arguments; device
    buffers are torch CUDA tensors or raw integer addresses, ``stream`` a
    ``torch.cuda.Stream``/raw handle/None for the current stream);
  * convenience wrappers (``sobel_binarize``, ``hough_accumulate``,
    ``hough_peaks``, ``detect_batch``, ``detect_batch_host``) that allocate the
    outputs with torch and call the ABI.

Every step of the path runs in the CUDA kernels of libld.so.  There is no CPU
fallback: if the library is missing or the device is not sm_100 the call
raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LD_LIB", os.path.join(HERE, "libld.so"))  # LD_LIB: dev override

LD_OK, LD_ERR_INVALID_ARG, LD_ERR_RANGE, LD_ERR_WORKSPACE, LD_ERR_UNSUPPORTED, LD_ERR_CUDA = range(6)
LD_MAX_DIM, LD_MAX_THETA, LD_MAX_K = 16384, 2048, 1024


class LdError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__("%s: %s" % (_STATUS.get(status, "LD_ERR_%d" % status), detail))
        self.status = status


_STATUS = {0: "LD_OK", 1: "LD_ERR_INVALID_ARG", 2: "LD_ERR_RANGE", 3: "LD_ERR_WORKSPACE",
           4: "LD_ERR_UNSUPPORTED", 5: "LD_ERR_CUDA"}


class ld_image(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("pitch", ctypes.c_int64), ("frame_stride", ctypes.c_int64),
                ("batch", ctypes.c_int32), ("row_begin", ctypes.c_int32),
                ("row_end", ctypes.c_int32)]


class ld_peak(ctypes.Structure):
    _fields_ = [("theta_bin", ctypes.c_int32), ("rho_bin", ctypes.c_int32),
                ("votes", ctypes.c_uint32)]


PEAK_DTYPE = np.dtype([("theta_bin", "<i4"), ("rho_bin", "<i4"), ("votes", "<u4")])

LD_FLAG_ZERO_PAD, LD_FLAG_CLAMP_255 = 1, 2
LD_VOTE_PLAIN, LD_VOTE_NO_CLUSTER = 1, 2
LD_PEAKS_DENSE, LD_PEAKS_FORCE_STREAM, LD_PEAKS_FORCE_TILE, LD_PEAKS_FORCE_BAND = 1, 2, 4, 8

EXPORTS = ["ld_rho_offset", "ld_sobel_binarize", "ld_sobel_binarize_ex", "ld_hough_accumulate",
           "ld_hough_hint_bytes", "ld_hough_accumulate_hint", "ld_hough_peaks_hinted",
           "ld_hough_hint_from_acc", "ld_hough_accumulate_f64", "ld_hough_accumulate_opt", "ld_hough_peaks_opt",
           "ld_edge_bitmask_words", "ld_edges_to_bitmask", "ld_bitmask_to_edges",
           "ld_merge_peak_lists",
           "ld_hough_peaks_workspace_bytes", "ld_hough_peaks", "ld_hough_peaks_ex",
           "ld_hough_peaks_nms_workspace_bytes", "ld_hough_peaks_nms", "ld_peak_lines",
           "ld_extract_segments",
           "ld_detect_workspace_bytes",
           "ld_detect_batch", "ld_detect_batch_ex", "ld_detect_host_workspace_bytes", "ld_detect_batch_host",
           "ld_bench_smem_atomics", "ld_device_sm_count", "ld_device_l2_bytes",
           "ld_status_string", "ld_last_error_detail", "ld_last_launch_count"]

_lib = None


def lib():
    """Load libld.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libld.so not found at %s; build it with "
                               "`python -m paper_2212_09460_b200.build`" % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, u32, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                ctypes.c_uint32, ctypes.c_size_t)
        IMG = ctypes.POINTER(ld_image)
        sig = {
            "ld_rho_offset": ([i32, i32], i32),
            "ld_sobel_binarize": ([P, IMG, i32, P, P, i64, P, P], ctypes.c_int),
            "ld_sobel_binarize_ex": ([P, IMG, i32, u32, P, P, i64, P, P], ctypes.c_int),
            "ld_hough_accumulate": ([P, P, i64, i32, i32, i32, i32, P, P, P, P], ctypes.c_int),
            "ld_hough_hint_bytes": ([i32, i32, i32, i32], sz),
            "ld_hough_accumulate_f64": ([P, P, i64, i32, i32, i32, i32, P, P, P, P], ctypes.c_int),
            "ld_hough_accumulate_hint": ([P, P, i64, i32, i32, i32, i32, P, P, P, P, sz, P],
                                         ctypes.c_int),
            "ld_hough_hint_from_acc": ([P, i32, i32, i32, i32, i32, P, sz, P], ctypes.c_int),
            "ld_hough_peaks_hinted": ([P, i32, i32, i32, i32, i32, u32, i32, P, sz, P, P, P, sz,
                                       P], ctypes.c_int),
            "ld_hough_peaks_workspace_bytes": ([i32, i32, i32, i32], sz),
            "ld_hough_peaks": ([P, i32, i32, i32, i32, i32, u32, i32, P, P, P, sz, P],
                               ctypes.c_int),
            "ld_hough_peaks_ex": ([P, i32, i32, i32, i32, i32, u32, i32, i32, i32, i32, P, P, P,
                                   sz, P], ctypes.c_int),
            "ld_hough_accumulate_opt": ([P, P, i64, i32, i32, i32, i32, P, P, u32, P, P, sz, P],
                                        ctypes.c_int),
            "ld_hough_peaks_opt": ([P, i32, i32, i32, i32, i32, u32, i32, i32, i32, i32, P, sz,
                                    u32, P, P, P, sz, P], ctypes.c_int),
            "ld_hough_peaks_nms_workspace_bytes": ([i32, i32, i32], sz),
            "ld_hough_peaks_nms": ([P, i32, i32, i32, i32, i32, u32, u32, u32, i32, P, P, P, sz,
                                    P], ctypes.c_int),
            "ld_peak_lines": ([P, P, i32, i32, i32, i32, i32, P, P, P, P, P], ctypes.c_int),
            "ld_extract_segments": ([P, IMG, P, P, i32, i32, P, P, i32, i32, i32, P, P, P],
                                    ctypes.c_int),
            "ld_detect_workspace_bytes": ([IMG, i32, i32, i32], sz),
            "ld_detect_batch": ([P, IMG, i32, i32, P, P, i32, i32, u32, i32, P, P, P, P, P, sz, P],
                                ctypes.c_int),
            "ld_detect_batch_ex": ([P, IMG, i32, u32, i32, P, P, i32, i32, u32, i32, P, P, P, P, P,
                                    sz, P], ctypes.c_int),
            "ld_detect_host_workspace_bytes": ([IMG, i32, i32, i32], sz),
            "ld_detect_batch_host": ([P, IMG, i32, i32, P, P, i32, i32, u32, i32, P, P, P, i32, P,
                                      sz, P], ctypes.c_int),
            "ld_bench_smem_atomics": ([i32, i32, i32, ctypes.POINTER(ctypes.c_uint64), P, P],
                                      ctypes.c_int),
            "ld_edge_bitmask_words": ([i32, i32], i64),
            "ld_edges_to_bitmask": ([P, P, i32, i32, i32, P, P], ctypes.c_int),
            "ld_bitmask_to_edges": ([P, i32, i32, P, P, i32, P, i64, P, P], ctypes.c_int),
            "ld_merge_peak_lists": ([P, P, i32, i32, i32, P, P, P], ctypes.c_int),
            "ld_device_sm_count": ([], i32),
            "ld_device_l2_bytes": ([], i64),
            "ld_status_string": ([ctypes.c_int], ctypes.c_char_p),
            "ld_last_error_detail": ([], ctypes.c_char_p),
            "ld_last_launch_count": ([], i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


# ----------------------------------------------------------------------------
# marshalling helpers
# ----------------------------------------------------------------------------
def _addr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError("cannot take the address of %r" % type(x))


def _host_i32(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return a


def _stream(s):
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _check(rc: int):
    if rc != LD_OK:
        raise LdError(rc, lib().ld_last_error_detail().decode())


def make_image(width, height, pitch=None, frame_stride=None, batch=1, row_begin=0,
               row_end=None) -> ld_image:
    pitch = width if pitch is None else pitch
    row_end = height if row_end is None else row_end
    if frame_stride is None:
        rb = max(row_begin - 1, 0)
        re = min(row_end + 1, height)
        frame_stride = (re - rb) * pitch
    return ld_image(width, height, pitch, frame_stride, batch, row_begin, row_end)


# ----------------------------------------------------------------------------
# C ABI, one-to-one
# ----------------------------------------------------------------------------
def ld_rho_offset(width: int, height: int) -> int:
    return int(lib().ld_rho_offset(width, height))


def ld_sobel_binarize(gray, img: ld_image, threshold, binary, edge_xy, edge_stride, edge_count,
                      stream=None):
    _check(lib().ld_sobel_binarize(_addr(gray), ctypes.byref(img), int(threshold), _addr(binary),
                                   _addr(edge_xy), int(edge_stride), _addr(edge_count),
                                   _stream(stream)))


def ld_sobel_binarize_ex(gray, img: ld_image, threshold, flags, binary, edge_xy, edge_stride,
                         edge_count, stream=None):
    _check(lib().ld_sobel_binarize_ex(_addr(gray), ctypes.byref(img), int(threshold), int(flags),
                                      _addr(binary), _addr(edge_xy), int(edge_stride),
                                      _addr(edge_count), _stream(stream)))


def ld_hough_accumulate(edge_xy, edge_count, edge_stride, batch, width, height, n_theta,
                        cos_q15, sin_q15, acc, stream=None):
    c, s = _host_i32(cos_q15), _host_i32(sin_q15)
    _check(lib().ld_hough_accumulate(_addr(edge_xy), _addr(edge_count), int(edge_stride),
                                     int(batch), int(width), int(height), int(n_theta),
                                     _addr(c), _addr(s), _addr(acc), _stream(stream)))


def ld_hough_accumulate_opt(edge_xy, edge_count, edge_stride, batch, width, height, n_theta,
                            cos_q15, sin_q15, flags, acc, hint=None, hint_bytes=0, stream=None):
    c, s = _host_i32(cos_q15), _host_i32(sin_q15)
    _check(lib().ld_hough_accumulate_opt(_addr(edge_xy), _addr(edge_count), int(edge_stride),
                                         int(batch), int(width), int(height), int(n_theta),
                                         _addr(c), _addr(s), int(flags), _addr(acc), _addr(hint),
                                         int(hint_bytes), _stream(stream)))


def ld_hough_accumulate_f64(edge_xy, edge_count, edge_stride, batch, width, height, n_theta,
                            cos_f64, sin_f64, acc, stream=None):
    c = np.ascontiguousarray(np.asarray(cos_f64, dtype=np.float64))
    s = np.ascontiguousarray(np.asarray(sin_f64, dtype=np.float64))
    _check(lib().ld_hough_accumulate_f64(_addr(edge_xy), _addr(edge_count), int(edge_stride),
                                         int(batch), int(width), int(height), int(n_theta),
                                         _addr(c), _addr(s), _addr(acc), _stream(stream)))


def hough_accumulate_f64(edges, counts, edge_stride, width, height, cos_f64, sin_f64,
                         stream=None):
    """SPEC float64 trig mode (ld_hough_accumulate_f64)."""
    import torch
    b = counts.shape[0]
    n_theta = len(cos_f64)
    n_rho = 2 * ld_rho_offset(width, height) + 1
    acc = torch.empty((b, n_theta, n_rho), dtype=torch.int32, device=counts.device)
    ld_hough_accumulate_f64(edges, counts, edge_stride, b, width, height, n_theta, cos_f64,
                            sin_f64, acc, stream)
    return acc


def ld_hough_hint_bytes(batch, width, height, n_theta) -> int:
    return int(lib().ld_hough_hint_bytes(batch, width, height, n_theta))


def ld_hough_accumulate_hint(edge_xy, edge_count, edge_stride, batch, width, height, n_theta,
                             cos_q15, sin_q15, acc, hint, hint_bytes, stream=None):
    c, s = _host_i32(cos_q15), _host_i32(sin_q15)
    _check(lib().ld_hough_accumulate_hint(_addr(edge_xy), _addr(edge_count), int(edge_stride),
                                          int(batch), int(width), int(height), int(n_theta),
                                          _addr(c), _addr(s), _addr(acc), _addr(hint),
                                          int(hint_bytes), _stream(stream)))


def ld_hough_hint_from_acc(acc, batch, n_theta, n_rho, cand_row_begin, cand_row_end, hint,
                           hint_bytes, stream=None):
    _check(lib().ld_hough_hint_from_acc(_addr(acc), int(batch), int(n_theta), int(n_rho),
                                        int(cand_row_begin), int(cand_row_end), _addr(hint),
                                        int(hint_bytes), _stream(stream)))


def ld_hough_peaks_hinted(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, k, hint,
                          hint_bytes, peaks, n_peaks, workspace, workspace_bytes, stream=None):
    _check(lib().ld_hough_peaks_hinted(_addr(acc), int(batch), int(n_theta), int(n_rho),
                                       int(half_theta), int(half_rho), int(min_votes), int(k),
                                       _addr(hint), int(hint_bytes), _addr(peaks),
                                       _addr(n_peaks), _addr(workspace), int(workspace_bytes),
                                       _stream(stream)))


def ld_hough_peaks_workspace_bytes(batch, n_theta, n_rho, k) -> int:
    return int(lib().ld_hough_peaks_workspace_bytes(batch, n_theta, n_rho, k))


def ld_hough_peaks(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, k, peaks,
                   n_peaks, workspace, workspace_bytes, stream=None):
    _check(lib().ld_hough_peaks(_addr(acc), int(batch), int(n_theta), int(n_rho),
                                int(half_theta), int(half_rho), int(min_votes), int(k),
                                _addr(peaks), _addr(n_peaks), _addr(workspace),
                                int(workspace_bytes), _stream(stream)))


def ld_hough_peaks_ex(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, k,
                      cand_row_begin, cand_row_end, theta_offset, peaks, n_peaks, workspace,
                      workspace_bytes, stream=None):
    _check(lib().ld_hough_peaks_ex(_addr(acc), int(batch), int(n_theta), int(n_rho),
                                   int(half_theta), int(half_rho), int(min_votes), int(k),
                                   int(cand_row_begin), int(cand_row_end), int(theta_offset),
                                   _addr(peaks), _addr(n_peaks), _addr(workspace),
                                   int(workspace_bytes), _stream(stream)))


def ld_hough_peaks_opt(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, k,
                       cand_row_begin, cand_row_end, theta_offset, hint, hint_bytes, flags, peaks,
                       n_peaks, workspace, workspace_bytes, stream=None):
    _check(lib().ld_hough_peaks_opt(_addr(acc), int(batch), int(n_theta), int(n_rho),
                                    int(half_theta), int(half_rho), int(min_votes), int(k),
                                    int(cand_row_begin), int(cand_row_end), int(theta_offset),
                                    _addr(hint), int(hint_bytes), int(flags), _addr(peaks),
                                    _addr(n_peaks), _addr(workspace), int(workspace_bytes),
                                    _stream(stream)))


def ld_hough_peaks_nms_workspace_bytes(batch, n_theta, n_rho) -> int:
    return int(lib().ld_hough_peaks_nms_workspace_bytes(batch, n_theta, n_rho))


def ld_hough_peaks_nms(acc, batch, n_theta, n_rho, half_theta, half_rho, min_votes, ratio_num,
                       ratio_den, k, peaks, n_peaks, workspace, workspace_bytes, stream=None):
    _check(lib().ld_hough_peaks_nms(_addr(acc), int(batch), int(n_theta), int(n_rho),
                                    int(half_theta), int(half_rho), int(min_votes),
                                    int(ratio_num), int(ratio_den), int(k), _addr(peaks),
                                    _addr(n_peaks), _addr(workspace), int(workspace_bytes),
                                    _stream(stream)))


def ld_peak_lines(peaks, n_peaks, batch, k, width, height, n_theta, cos_q15, sin_q15, lines,
                  hit, stream=None):
    c, s = _host_i32(cos_q15), _host_i32(sin_q15)
    _check(lib().ld_peak_lines(_addr(peaks), _addr(n_peaks), int(batch), int(k), int(width),
                               int(height), int(n_theta), _addr(c), _addr(s), _addr(lines),
                               _addr(hit), _stream(stream)))


def ld_extract_segments(binary, img: ld_image, peaks, n_peaks, k, n_theta, cos_q15, sin_q15,
                        fill_gap, min_len, max_segments, segments, n_segments, stream=None):
    c, s = _host_i32(cos_q15), _host_i32(sin_q15)
    _check(lib().ld_extract_segments(_addr(binary), ctypes.byref(img), _addr(peaks),
                                     _addr(n_peaks), int(k), int(n_theta), _addr(c), _addr(s),
                                     int(fill_gap), int(min_len), int(max_segments),
                                     _addr(segments), _addr(n_segments), _stream(stream)))


def ld_detect_workspace_bytes(img: ld_image, n_theta, k, acc_in_workspace) -> int:
    return int(lib().ld_detect_workspace_bytes(ctypes.byref(img), n_theta, k,
                                               int(bool(acc_in_workspace))))


def ld_detect_batch(gray, img: ld_image, threshold, n_theta, cos_q15, sin_q15, half_theta,
                    half_rho, min_votes, k, peaks, n_peaks, edge_count, acc, workspace,
                    workspace_bytes, stream=None):
    c, s = _host_i32(cos_q15), _host_i32(sin_q15)
    _check(lib().ld_detect_batch(_addr(gray), ctypes.byref(img), int(threshold), int(n_theta),
                                 _addr(c), _addr(s), int(half_theta), int(half_rho),
                                 int(min_votes), int(k), _addr(peaks), _addr(n_peaks),
                                 _addr(edge_count), _addr(acc), _addr(workspace),
                                 int(workspace_bytes), _stream(stream)))


def ld_detect_batch_ex(gray, img: ld_image, threshold, flags, n_theta, cos_q15, sin_q15,
                       half_theta, half_rho, min_votes, k, peaks, n_peaks, edge_count, acc,
                       workspace, workspace_bytes, stream=None):
    c, s = _host_i32(cos_q15), _host_i32(sin_q15)
    _check(lib().ld_detect_batch_ex(_addr(gray), ctypes.byref(img), int(threshold), int(flags),
                                    int(n_theta), _addr(c), _addr(s), int(half_theta),
                                    int(half_rho), int(min_votes), int(k), _addr(peaks),
                                    _addr(n_peaks), _addr(edge_count), _addr(acc),
                                    _addr(workspace), int(workspace_bytes), _stream(stream)))


def ld_detect_host_workspace_bytes(img: ld_image, n_theta, k, chunk_frames) -> int:
    return int(lib().ld_detect_host_workspace_bytes(ctypes.byref(img), n_theta, k, chunk_frames))


def ld_detect_batch_host(gray_host, img: ld_image, threshold, n_theta, cos_q15, sin_q15,
                         half_theta, half_rho, min_votes, k, peaks_host, n_peaks_host,
                         edge_count_host, chunk_frames, workspace, workspace_bytes, stream=None):
    c, s = _host_i32(cos_q15), _host_i32(sin_q15)
    _check(lib().ld_detect_batch_host(_addr(gray_host), ctypes.byref(img), int(threshold),
                                      int(n_theta), _addr(c), _addr(s), int(half_theta),
                                      int(half_rho), int(min_votes), int(k), _addr(peaks_host),
                                      _addr(n_peaks_host), _addr(edge_count_host),
                                      int(chunk_frames), _addr(workspace), int(workspace_bytes),
                                      _stream(stream)))


def ld_bench_smem_atomics(mode, iters, blocks_per_sm, scratch, stream=None) -> int:
    n = ctypes.c_uint64(0)
    _check(lib().ld_bench_smem_atomics(int(mode), int(iters), int(blocks_per_sm),
                                       ctypes.byref(n), _addr(scratch), _stream(stream)))
    return int(n.value)


def ld_edge_bitmask_words(width, rows) -> int:
    return int(lib().ld_edge_bitmask_words(int(width), int(rows)))


def ld_edges_to_bitmask(edge_xy, edge_count, width, row_begin, rows, bits, stream=None):
    _check(lib().ld_edges_to_bitmask(_addr(edge_xy), _addr(edge_count), int(width),
                                     int(row_begin), int(rows), _addr(bits), _stream(stream)))


def ld_bitmask_to_edges(bits, width, block_row_begin, block_rows, block_stride_rows, edge_xy,
                        edge_capacity, edge_count, stream=None):
    rb, rr = _host_i32(block_row_begin), _host_i32(block_rows)
    _check(lib().ld_bitmask_to_edges(_addr(bits), int(width), int(len(rb)), _addr(rb),
                                     _addr(rr), int(block_stride_rows), _addr(edge_xy),
                                     int(edge_capacity), _addr(edge_count), _stream(stream)))


def ld_merge_peak_lists(peaks, n_peaks, n_lists, k, n_rho, out, n_out, stream=None):
    _check(lib().ld_merge_peak_lists(_addr(peaks), _addr(n_peaks), int(n_lists), int(k),
                                     int(n_rho), _addr(out), _addr(n_out), _stream(stream)))


def ld_device_sm_count() -> int:
    return int(lib().ld_device_sm_count())


def ld_device_l2_bytes() -> int:
    return int(lib().ld_device_l2_bytes())


def ld_last_launch_count() -> int:
    return int(lib().ld_last_launch_count())


# ----------------------------------------------------------------------------
# convenience wrappers (torch tensors in, torch tensors out)
# ----------------------------------------------------------------------------
def _round_up(v, a):
    return (v + a - 1) // a * a


def pitched(gray):
    """uint8 CUDA tensor [B][H][W] -> (tensor whose rows are 16-byte padded, pitch)."""
    import torch
    b, h, w = gray.shape
    pitch = _round_up(w, 16)
    if pitch == w and gray.is_contiguous():
        return gray, pitch
    out = torch.zeros((b, h, pitch), dtype=torch.uint8, device=gray.device)
    out[:, :, :w] = gray
    return out, pitch


def sobel_binarize(gray, threshold: int, want_binary=True, want_edges=True, stream=None,
                   flags: int = 0):
    """gray: uint8 CUDA [B][H][W] (whole frames).  Returns (binary [B][H][W] or
    None, edges [B][edge_stride] or None, counts [B], edge_stride).  flags:
    LD_FLAG_ZERO_PAD / LD_FLAG_CLAMP_255 (ld_sobel_binarize_ex)."""
    import torch
    b, h, w = gray.shape
    g, pitch = pitched(gray)
    img = make_image(w, h, pitch, h * pitch, b)
    dev = gray.device
    stride = _round_up(max(h * (w if flags & LD_FLAG_ZERO_PAD else max(w - 2, 0)), 1), 4)
    binary = torch.empty((b, h, pitch), dtype=torch.uint8, device=dev) if want_binary else None
    edges = torch.empty((b, stride), dtype=torch.int32, device=dev) if want_edges else None
    counts = torch.empty((b,), dtype=torch.int32, device=dev)
    ld_sobel_binarize_ex(g, img, threshold, flags, binary, edges, stride, counts, stream)
    if binary is not None:
        binary = binary[:, :, :w]
    return binary, edges, counts, stride


def hough_accumulate(edges, counts, edge_stride, width, height, cos_q15, sin_q15, stream=None,
                     want_hint=False, flags=0):
    """Returns acc, or (acc, hint) with want_hint (ld_hough_accumulate_hint).
    flags: LD_VOTE_PLAIN (ld_hough_accumulate_opt)."""
    import torch
    b = counts.shape[0]
    n_theta = len(cos_q15)
    n_rho = 2 * ld_rho_offset(width, height) + 1
    acc = torch.empty((b, n_theta, n_rho), dtype=torch.int32, device=counts.device)
    hint, hb = None, 0
    if want_hint:
        hb = ld_hough_hint_bytes(b, width, height, n_theta)
        hint = torch.empty((hb,), dtype=torch.uint8, device=counts.device)
    ld_hough_accumulate_opt(edges, counts, edge_stride, b, width, height, n_theta, cos_q15,
                            sin_q15, flags, acc, hint, hb, stream)
    return (acc, hint) if want_hint else acc


def hint_from_acc(acc, width, height, cand_rows=None, stream=None):
    """The peak hint of an existing accumulator (ld_hough_hint_from_acc):
    acc int32 CUDA [B][n_theta][n_rho] of a width x height image (n_rho =
    2 ld_rho_offset + 1); cand_rows=(begin, end) limits the recorded keys."""
    import torch
    b, n_theta, n_rho = acc.shape
    hb = ld_hough_hint_bytes(b, width, height, n_theta)
    hint = torch.empty((hb,), dtype=torch.uint8, device=acc.device)
    c0, c1 = cand_rows if cand_rows is not None else (0, n_theta)
    ld_hough_hint_from_acc(acc, b, n_theta, n_rho, c0, c1, hint, hb, stream)
    return hint


def hough_peaks(acc, half_theta, half_rho, min_votes, k, stream=None, cand_rows=None,
                theta_offset=0, hint=None, flags=0):
    """acc: int32 CUDA [B][n_theta][n_rho] (uint32 bits).  cand_rows=(begin, end)
    and theta_offset select ld_hough_peaks_ex (a theta slice of a larger
    accumulator); hint (from hough_accumulate(want_hint=True)) selects
    ld_hough_peaks_hinted; flags (LD_PEAKS_*) select ld_hough_peaks_opt."""
    import torch
    b, n_theta, n_rho = acc.shape
    ws_bytes = ld_hough_peaks_workspace_bytes(b, n_theta, n_rho, k)
    ws = torch.empty((max(ws_bytes, 16),), dtype=torch.uint8, device=acc.device)
    peaks = torch.empty((b, k, 3), dtype=torch.int32, device=acc.device)
    n_peaks = torch.empty((b,), dtype=torch.int32, device=acc.device)
    if flags or (hint is not None and (cand_rows is not None or theta_offset)):
        c0, c1 = cand_rows if cand_rows is not None else (0, n_theta)
        ld_hough_peaks_opt(acc, b, n_theta, n_rho, half_theta, half_rho, min_votes, k, c0, c1,
                           theta_offset, hint, 0 if hint is None else hint.numel(), flags, peaks,
                           n_peaks, ws, ws_bytes, stream)
    elif hint is not None:
        ld_hough_peaks_hinted(acc, b, n_theta, n_rho, half_theta, half_rho, min_votes, k, hint,
                              hint.numel(), peaks, n_peaks, ws, ws_bytes, stream)
    elif cand_rows is None and theta_offset == 0:
        ld_hough_peaks(acc, b, n_theta, n_rho, half_theta, half_rho, min_votes, k, peaks,
                       n_peaks, ws, ws_bytes, stream)
    else:
        c0, c1 = cand_rows if cand_rows is not None else (0, n_theta)
        ld_hough_peaks_ex(acc, b, n_theta, n_rho, half_theta, half_rho, min_votes, k, c0, c1,
                          theta_offset, peaks, n_peaks, ws, ws_bytes, stream)
    return peaks, n_peaks


class Detector:
    """Owns the device workspace for repeated ld_detect_batch calls on one shape."""

    def __init__(self, width, height, batch, n_theta, cos_q15, sin_q15, threshold, k,
                 half_theta, half_rho, min_votes=1, export_acc=False, device=None, flags=0):
        import torch
        self.flags = int(flags)
        self.device = torch.device("cuda") if device is None else device
        self.w, self.h, self.b = width, height, batch
        self.pitch = _round_up(width, 16)
        self.img = make_image(width, height, self.pitch, height * self.pitch, batch)
        self.n_theta, self.k = n_theta, k
        self.cos, self.sin = _host_i32(cos_q15), _host_i32(sin_q15)
        self.threshold, self.half_theta, self.half_rho = threshold, half_theta, half_rho
        self.min_votes = min_votes
        self.n_rho = 2 * ld_rho_offset(width, height) + 1
        self.ws_bytes = ld_detect_workspace_bytes(self.img, n_theta, k, not export_acc)
        self.ws = torch.empty((self.ws_bytes,), dtype=torch.uint8, device=self.device)
        self.peaks = torch.empty((batch, k, 3), dtype=torch.int32, device=self.device)
        self.n_peaks = torch.empty((batch,), dtype=torch.int32, device=self.device)
        self.counts = torch.empty((batch,), dtype=torch.int32, device=self.device)
        self.acc = (torch.empty((batch, n_theta, self.n_rho), dtype=torch.int32,
                                device=self.device) if export_acc else None)

    def __call__(self, gray, stream=None):
        """gray: uint8 CUDA [B][H][pitch] with pitch = round_up(W, 16).  Runs on
        the detector's device (the C ABI uses the current device), on `stream`
        or that device's current stream."""
        import torch
        with torch.cuda.device(self.device):
            if stream is None:
                stream = torch.cuda.current_stream(self.device)
            ld_detect_batch_ex(gray, self.img, self.threshold, self.flags, self.n_theta,
                               self.cos, self.sin, self.half_theta, self.half_rho,
                               self.min_votes, self.k, self.peaks, self.n_peaks, self.counts,
                               self.acc, self.ws, self.ws_bytes, stream)
        return self.peaks, self.n_peaks, self.counts, self.acc


class PipelinedDetector:
    """Batches in flight on several streams (the benchmark's serving mode).

    Each of `streams` slots owns a Detector (its own workspace and outputs)
    and a CUDA stream; submit() enqueues ld_detect_batch for one batch on the
    next slot, after the caller's current stream (so the input is ready), and
    returns that slot's (peaks, n_peaks, counts) tensors and a CUDA event that
    completes with them.  A slot is reused `streams` submissions later, which
    first waits for its previous batch (the stream order does it).  Step i's
    peak search then overlaps step i+1's Sobel on the GPU."""

    def __init__(self, width, height, batch, n_theta, cos_q15, sin_q15, threshold, k,
                 half_theta, half_rho, min_votes=1, streams=4, device=None, flags=0):
        import torch
        self.slots = []
        for _ in range(streams):
            det = Detector(width, height, batch, n_theta, cos_q15, sin_q15, threshold, k,
                           half_theta, half_rho, min_votes, False, device, flags)
            self.slots.append((det, torch.cuda.Stream(device=det.device)))
        self.next = 0

    def submit(self, gray):
        """gray: uint8 CUDA [B][H][pitch] (pitch = round_up(W, 16)); must stay
        unmodified until the returned event completes."""
        import torch
        det, st = self.slots[self.next]
        self.next = (self.next + 1) % len(self.slots)
        st.wait_stream(torch.cuda.current_stream(det.device))
        # the caller may drop `gray` right away: keep the caching allocator
        # from handing its memory to another stream while `st` still reads it
        gray.record_stream(st)
        det(gray, st)
        ev = torch.cuda.Event()
        ev.record(st)
        return det.peaks, det.n_peaks, det.counts, ev


def detect_batch(gray, threshold, cos_q15, sin_q15, half_theta, half_rho, min_votes, k,
                 export_acc=True, stream=None):
    b, h, w = gray.shape
    g, pitch = pitched(gray)
    det = Detector(w, h, b, len(cos_q15), cos_q15, sin_q15, threshold, k, half_theta, half_rho,
                   min_votes, export_acc, gray.device)
    return det(g, stream)


class HostDetector:
    """ld_detect_batch_host: host (pinned) frames in, host peaks out."""

    def __init__(self, width, height, batch, n_theta, cos_q15, sin_q15, threshold, k,
                 half_theta, half_rho, min_votes=1, chunk_frames=32, device=None):
        import torch
        self.device = torch.device("cuda") if device is None else device
        self.pitch = _round_up(width, 16)
        self.img = make_image(width, height, self.pitch, height * self.pitch, batch)
        self.n_theta, self.k, self.chunk = n_theta, k, chunk_frames
        self.cos, self.sin = _host_i32(cos_q15), _host_i32(sin_q15)
        self.threshold, self.half_theta, self.half_rho = threshold, half_theta, half_rho
        self.min_votes = min_votes
        self.ws_bytes = ld_detect_host_workspace_bytes(self.img, n_theta, k, chunk_frames)
        self.ws = torch.empty((self.ws_bytes,), dtype=torch.uint8, device=self.device)
        self.peaks = torch.empty((batch, k, 3), dtype=torch.int32).pin_memory()
        self.n_peaks = torch.empty((batch,), dtype=torch.int32).pin_memory()
        self.counts = torch.empty((batch,), dtype=torch.int32).pin_memory()

    def __call__(self, gray_host, stream=None):
        """Runs on the detector's device (the C ABI uses the current device),
        on `stream` or that device's current stream."""
        import torch
        with torch.cuda.device(self.device):
            if stream is None:
                stream = torch.cuda.current_stream(self.device)
            ld_detect_batch_host(gray_host, self.img, self.threshold, self.n_theta, self.cos,
                                 self.sin, self.half_theta, self.half_rho, self.min_votes,
                                 self.k, self.peaks, self.n_peaks, self.counts, self.chunk,
                                 self.ws, self.ws_bytes, stream)
        return self.peaks, self.n_peaks, self.counts


# ----------------------------------------------------------------------------
# lanes module (NEXT 3) convenience wrappers
# ----------------------------------------------------------------------------
def hough_peaks_nms(acc, half_theta, half_rho, min_votes, k, ratio=(0, 1), stream=None):
    """Greedy NMS (ld_hough_peaks_nms); ratio = (num, den): votes >= num/den * max."""
    import torch
    b, n_theta, n_rho = acc.shape
    wsb = ld_hough_peaks_nms_workspace_bytes(b, n_theta, n_rho)
    ws = torch.empty((wsb,), dtype=torch.uint8, device=acc.device)
    peaks = torch.empty((b, k, 3), dtype=torch.int32, device=acc.device)
    n_peaks = torch.empty((b,), dtype=torch.int32, device=acc.device)
    ld_hough_peaks_nms(acc, b, n_theta, n_rho, half_theta, half_rho, min_votes, ratio[0],
                       ratio[1], k, peaks, n_peaks, ws, wsb, stream)
    return peaks, n_peaks


def peak_lines(peaks, n_peaks, width, height, cos_q15, sin_q15, stream=None):
    """Returns (lines int32 [B][k][4], hit int32 [B][k])."""
    import torch
    b, k, _ = peaks.shape
    lines = torch.zeros((b, k, 4), dtype=torch.int32, device=peaks.device)
    hit = torch.empty((b, k), dtype=torch.int32, device=peaks.device)
    ld_peak_lines(peaks, n_peaks, b, k, width, height, len(cos_q15), cos_q15, sin_q15, lines, hit,
                  stream)
    return lines, hit


def extract_segments(binary, peaks, n_peaks, cos_q15, sin_q15, fill_gap=20, min_len=40,
                     max_segments=64, width=None, stream=None):
    """binary: contiguous uint8 CUDA [B][H][pitch] (pitch >= width; width
    defaults to pitch).  Returns (segments int32 [B][k][max_segments][4],
    n_segments int32 [B][k])."""
    import torch
    b, h, pitch = binary.shape
    k = peaks.shape[1]
    width = pitch if width is None else width
    img = make_image(width, h, pitch, h * pitch, b)
    segs = torch.zeros((b, k, max_segments, 4), dtype=torch.int32, device=binary.device)
    nseg = torch.empty((b, k), dtype=torch.int32, device=binary.device)
    ld_extract_segments(binary, img, peaks, n_peaks, k, len(cos_q15), cos_q15, sin_q15, fill_gap,
                        min_len, max_segments, segs, nseg, stream)
    return segs, nseg
