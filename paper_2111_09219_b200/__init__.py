"""paper_2111_09219_b200 — B200-native fully-on-GPU baseline-JPEG decoder.

Python mirror of the reference's decode API (pjpeg, proj/include/pjpeg/
pipeline.hpp) over the C-ABI in ``include/pjg.h`` (``libpjg.so``):

    DecodeConfig, DecodeSuccess, DecodeFailure, Error, Errc,
    decode_single, decode_batch, upsample_and_convert, planes_checksum

plus the staged device pipeline (:class:`Decoder`, :class:`Batch`) used by the
benchmark and the parity taps.  All decoding runs in the sm_100a kernels of
``libpjg.so``; there is no CPU fallback — importing works without a GPU, but
every decode call fails loudly if the library or the device is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Errc", "Error", "DecodeConfig", "OutputColorspace", "ImagePlanes", "Plane", "RgbImage",
    "StageTimings", "DecodeSuccess", "DecodeFailure", "decode_single", "decode_batch",
    "upsample_and_convert", "planes_checksum", "Decoder", "Batch", "lib", "LIB_PATH",
    "decode_to_tensors",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PJG_LIB") or os.path.join(HERE, "libpjg.so")  # PJG_LIB: A/B experiments


class Errc(enum.IntEnum):
    """pjpeg::Errc (common.hpp:26-38); the C-ABI status is value + 1."""
    MalformedStuffing = 0
    EmptyScan = 1
    OutOfBits = 2
    UnsupportedFeature = 3
    MalformedHeader = 4
    MissingTable = 5
    OversubscribedCode = 6
    InvalidCode = 7
    ConsistencyFailure = 8
    EmptyCorpus = 9
    IoError = 10


class Error(RuntimeError):
    """pjpeg::Error (common.hpp:57-66).  ``code`` is an :class:`Errc` for
    decode errors, or None for runtime failures (CUDA, arguments)."""

    def __init__(self, status: int, message: str = ""):
        self.status = int(status)
        self.code = Errc(status - 1) if 1 <= status <= 11 else None
        name = self.code.name if self.code is not None else _status_name(status)
        super().__init__(f"{name}: {message}" if message else name)


class OutputColorspace(enum.IntEnum):
    """pjpeg::OutputColorspace (pipeline.hpp:34)."""
    YCbCrPlanes = 0
    RGBInterleaved = 1
    Grayscale = 2


@dataclass
class DecodeConfig:
    """pjpeg::DecodeConfig (pipeline.hpp:36-41).  ``worker_count`` is accepted
    for signature parity; the GPU sizes its own grids."""
    subsequence_bits: int = 1024
    sequence_length_b: int = 256
    worker_count: int = 1
    output_colorspace: OutputColorspace = OutputColorspace.YCbCrPlanes
    # extension: decode restart intervals (DRI + RSTn); False = the reference's
    # UnsupportedFeature for DRI != 0 (parser.hpp:299-302)
    restart_intervals: bool = False


@dataclass
class Plane:
    width: int
    height: int
    samples: np.ndarray  # uint8 [height, width]

    def at(self, x, y):
        return int(self.samples[y, x])


@dataclass
class ImagePlanes:
    """pjpeg::ImagePlanes (transform.hpp:38-51)."""
    width: int = 0
    height: int = 0
    h_max: int = 1
    v_max: int = 1
    planes: list = field(default_factory=list)


@dataclass
class RgbImage:
    """pjpeg::RgbImage (pipeline.hpp:64-69); pixels HxWx3 (or HxW gray)."""
    width: int = 0
    height: int = 0
    pixels: np.ndarray | None = None
    channels: int = 3


@dataclass
class StageTimings:
    """Device stage times in ms (CUDA events).  Field names follow
    pjpeg::StageTimings (pipeline.hpp:44-62) where stages correspond."""
    upload: float = 0.0
    unstuff: float = 0.0
    sync: float = 0.0
    scan: float = 0.0
    write: float = 0.0
    idct: float = 0.0
    download: float = 0.0

    def total(self):
        return self.upload + self.unstuff + self.sync + self.scan + self.write + self.idct + self.download


@dataclass
class DecodeSuccess:
    planes: ImagePlanes
    timings: StageTimings
    compressed_bytes: int = 0


@dataclass
class DecodeFailure:
    code: Errc
    message: str = ""


# ---------------------------------------------------------------- ctypes --
class _Config(C.Structure):
    _fields_ = [("subsequence_bits", C.c_uint64), ("sequence_length_b", C.c_uint32),
                ("output", C.c_uint32), ("restart_intervals", C.c_uint32), ("reserved", C.c_uint32)]


class _Info(C.Structure):
    _fields_ = [("width", C.c_uint32), ("height", C.c_uint32), ("channels", C.c_uint32),
                ("num_components", C.c_uint32), ("plane_width", C.c_uint32 * 3),
                ("plane_height", C.c_uint32 * 3), ("h_max", C.c_uint32), ("v_max", C.c_uint32),
                ("mcus_x", C.c_uint32), ("mcus_y", C.c_uint32), ("output_bytes", C.c_uint64),
                ("compressed_bytes", C.c_uint64), ("data_units", C.c_uint64)]


class _SyncEntry(C.Structure):
    _fields_ = [("p", C.c_uint64), ("n", C.c_uint64), ("c", C.c_uint32), ("z", C.c_uint32),
                ("divergent", C.c_uint32), ("pad", C.c_uint32)]


_lib = None
_lib_lock = threading.Lock()
u8p = C.POINTER(C.c_uint8)


def lib():
    """Loads libpjg.so (built in-tree by ``make -C paper_2111_09219_b200/csrc``
    or ``__graft_entry__.build()``); raises if it is missing."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                                   "`make -C paper_2111_09219_b200/csrc` (no CPU fallback exists)")
            L = C.CDLL(LIB_PATH)
            L.pjg_status_name.restype = C.c_char_p
            L.pjg_last_error.restype = C.c_char_p
            L.pjg_batch_device_output.restype = C.c_void_p
            L.pjg_batch_output_bytes.restype = C.c_uint64
            L.pjg_ctx_stream.restype = C.c_void_p
            L.pjg_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
            L.pjg_ctx_destroy.argtypes = [C.c_void_p]
            L.pjg_last_error.argtypes = [C.c_void_p]
            L.pjg_ctx_stream.argtypes = [C.c_void_p]
            L.pjg_batch_create.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(u8p),
                                           C.POINTER(C.c_size_t), C.POINTER(_Config),
                                           C.POINTER(C.c_void_p)]
            L.pjg_batch_create_blob.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t,
                                                C.POINTER(C.c_uint64), C.POINTER(C.c_size_t),
                                                C.POINTER(_Config), C.POINTER(C.c_void_p)]
            L.pjg_batch_create_device.argtypes = L.pjg_batch_create_blob.argtypes
            for fn in ("pjg_batch_upload", "pjg_batch_decode"):
                getattr(L, fn).argtypes = [C.c_void_p]
            L.pjg_batch_synchronize.argtypes = [C.c_void_p, C.c_void_p]
            L.pjg_batch_download.argtypes = [C.c_void_p, C.POINTER(u8p), C.POINTER(C.c_size_t)]
            L.pjg_batch_download_all.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
            L.pjg_batch_download_all_async.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
            L.pjg_batch_output_offset.argtypes = [C.c_void_p, C.c_size_t]
            L.pjg_batch_output_offset.restype = C.c_uint64
            L.pjg_batch_info.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(_Info)]
            L.pjg_batch_device_output.argtypes = [C.c_void_p, C.c_size_t]
            L.pjg_batch_copy_outputs.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
            L.pjg_batch_scan_bits.argtypes = [C.c_void_p]
            L.pjg_batch_scan_bits.restype = C.c_uint64
            L.pjg_batch_kernel_launches.argtypes = [C.c_void_p]
            L.pjg_batch_kernel_launches.restype = C.c_uint32
            L.pjg_batch_output_bytes.argtypes = [C.c_void_p]
            L.pjg_batch_stage_times.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
            L.pjg_batch_sync_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
            L.pjg_batch_destroy.argtypes = [C.c_void_p]
            L.pjg_batch_dump_coefficients.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p,
                                                      C.c_size_t]
            L.pjg_batch_dump_sync_states.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                                     C.POINTER(C.c_size_t)]
            L.pjg_batch_dump_segment.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                                 C.POINTER(C.c_size_t)]
            L.pjg_inspect.argtypes = [C.c_void_p, C.c_size_t, C.c_uint32, C.POINTER(_Info)]
            L.pjg_upsample_and_convert.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                                   C.POINTER(u8p), u8p]
            L.pjg_debug_huff_decode.argtypes = [u8p, u8p, C.c_size_t, C.POINTER(C.c_uint16),
                                                C.c_size_t, C.POINTER(C.c_uint32)]
            L.pjg_debug_fast_entry.argtypes = [u8p, u8p, C.c_size_t, C.c_int, C.POINTER(C.c_uint32),
                                               C.c_size_t, C.POINTER(C.c_uint32)]
            _lib = L
        return _lib


EXPORTED_SYMBOLS = [
    "pjg_ctx_create", "pjg_ctx_destroy", "pjg_last_error", "pjg_status_name", "pjg_default_config",
    "pjg_ctx_stream", "pjg_inspect", "pjg_inspect_header", "pjg_decode", "pjg_decode_batch", "pjg_batch_create",
    "pjg_batch_create_blob", "pjg_batch_create_device", "pjg_batch_upload", "pjg_batch_decode", "pjg_batch_synchronize", "pjg_batch_download",
    "pjg_batch_info", "pjg_batch_device_output", "pjg_batch_copy_outputs", "pjg_batch_scan_bits", "pjg_batch_kernel_launches", "pjg_batch_download_all", "pjg_batch_download_all_async", "pjg_batch_output_offset", "pjg_batch_output_bytes", "pjg_batch_stage_times",
    "pjg_batch_sync_stats", "pjg_batch_destroy", "pjg_batch_dump_coefficients",
    "pjg_batch_dump_sync_states", "pjg_batch_dump_segment", "pjg_upsample_and_convert",
    "pjg_debug_huff_decode", "pjg_debug_fast_entry",
]


def _status_name(st: int) -> str:
    try:
        return lib().pjg_status_name(int(st)).decode()
    except Exception:  # pragma: no cover - library missing
        return f"status {st}"


def _cfg(config: DecodeConfig | None, output=None) -> _Config:
    config = config or DecodeConfig()
    out = int(config.output_colorspace if output is None else output)
    return _Config(int(config.subsequence_bits), int(config.sequence_length_b), out,
                   1 if config.restart_intervals else 0, 0)


# ------------------------------------------------------------ staged API --
class Decoder:
    """One pjg context = one (host thread, GPU) pair with its own stream."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        st = lib().pjg_ctx_create(int(device), C.byref(self._h))
        if st:
            raise Error(st, "pjg_ctx_create failed (is a CUDA device visible?)")
        self.device = device

    @property
    def handle(self):
        return self._h

    def last_error(self) -> str:
        return lib().pjg_last_error(self._h).decode()

    def stream(self) -> int:
        return int(lib().pjg_ctx_stream(self._h) or 0)

    def close(self):
        if self._h:
            lib().pjg_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def batch(self, files, config: DecodeConfig | None = None, output=None, device_plan=False) -> "Batch":
        return Batch(self, files, config, output, device_plan)


class Batch:
    """A planned batch on the device: create → upload → decode → synchronize
    → download / taps.  ``files`` is a list of bytes-like objects, or a tuple
    (blob: np.uint8 array, offsets, sizes) for files laid out contiguously
    (e.g. in pinned host memory) so the upload is one copy.  ``device_plan``:
    plan on the device (pjg_batch_create_device: header parse, tables and
    layout as kernels; whole files uploaded)."""

    def __init__(self, dec: Decoder, files, config=None, output=None, device_plan=False):
        self.dec = dec
        self.config = config or DecodeConfig()
        blob_args = None
        if isinstance(files, tuple):
            # one caller allocation: (blob uint8 array, offsets, sizes)
            blob, offsets, sizes = files
            blob = np.asarray(blob, np.uint8).reshape(-1)
            self._keep = [blob]
            n = len(sizes)
            oa = np.ascontiguousarray(offsets, np.uint64)
            sa = np.ascontiguousarray(sizes, np.uint64)
            self._keep += [oa, sa]
            blob_args = (C.c_void_p(blob.ctypes.data), blob.size, n,
                         oa.ctypes.data_as(C.POINTER(C.c_uint64)),
                         sa.ctypes.data_as(C.POINTER(C.c_size_t)))
        elif device_plan:  # one contiguous copy of the files
            arrs = [np.frombuffer(f, np.uint8) if not isinstance(f, np.ndarray) else f for f in files]
            sizes = np.array([a.size for a in arrs], np.uint64)
            offs = np.zeros(len(arrs), np.uint64)
            if len(arrs):
                offs[1:] = np.cumsum(sizes)[:-1]
            blob = np.concatenate(arrs) if arrs else np.zeros(1, np.uint8)
            self._keep = [blob, offs, sizes]
            n = len(arrs)
            blob_args = (C.c_void_p(blob.ctypes.data), blob.size, n,
                         offs.ctypes.data_as(C.POINTER(C.c_uint64)),
                         sizes.ctypes.data_as(C.POINTER(C.c_size_t)))
        else:
            self._keep = [np.frombuffer(f, np.uint8) if not isinstance(f, np.ndarray) else f
                          for f in files]
            n = len(self._keep)
            ptrs = (u8p * n)(*[a.ctypes.data_as(u8p) for a in self._keep])
            szs = (C.c_size_t * n)(*[a.size for a in self._keep])
        self.n = n
        self._h = C.c_void_p()
        cfg = _cfg(self.config, output)
        self.output = cfg.output
        if blob_args is not None:
            fn = lib().pjg_batch_create_device if device_plan else lib().pjg_batch_create_blob
            st = fn(dec.handle, *blob_args, C.byref(cfg), C.byref(self._h))
        else:
            st = lib().pjg_batch_create(dec.handle, n, ptrs, szs, C.byref(cfg), C.byref(self._h))
        if st:
            raise Error(st, dec.last_error())
        self._infos = None

    @property
    def infos(self):
        """Per-image geometry (fetched lazily: the pipelined host path never needs it)."""
        if self._infos is None:
            self._infos, self.header_status = [], []
            for i in range(self.n):
                inf = _Info()
                self.header_status.append(lib().pjg_batch_info(self._h, i, C.byref(inf)))
                self._infos.append(inf)
        return self._infos

    def _check(self, st):
        if st:
            raise Error(st, self.dec.last_error())

    def upload(self):
        self._check(lib().pjg_batch_upload(self._h))
        return self

    def decode(self):
        self._check(lib().pjg_batch_decode(self._h))
        return self

    def synchronize(self) -> np.ndarray:
        out = np.zeros(self.n, np.int32)
        self._check(lib().pjg_batch_synchronize(self._h, out.ctypes.data_as(C.c_void_p)))
        self.status = out
        return out

    def run(self) -> np.ndarray:
        return self.upload().decode().synchronize()

    def scan_bits(self) -> int:
        """Unstuffed entropy-coded bits of the decoded images (after synchronize)."""
        return int(lib().pjg_batch_scan_bits(self._h))

    def kernel_launches(self) -> int:
        """Kernels one decode() of this batch launches."""
        return int(lib().pjg_batch_kernel_launches(self._h))

    def output_bytes(self) -> int:
        return int(lib().pjg_batch_output_bytes(self._h))

    def device_output(self, i) -> int:
        return int(lib().pjg_batch_device_output(self._h, i) or 0)

    def tensors(self):
        """The decoded images as CUDA uint8 torch tensors on the decoder's device
        ((H, W, 3) RGB, (H, W) gray, flat planes otherwise), filled by
        device-to-device copies ordered after the decode; torch's current
        stream waits for them.  Failed images get None."""
        import torch
        dev = torch.device("cuda", self.dec.device)
        outs, ptrs, caps = [], [], []
        for i, inf in enumerate(self.infos):
            nb = int(inf.output_bytes)
            if (getattr(self, "status", None) is not None and self.status[i] != 0) or nb == 0:
                outs.append(None)
                ptrs.append(None)
                caps.append(0)
                continue
            if self.output == int(OutputColorspace.RGBInterleaved) and inf.channels == 3:
                t = torch.empty((inf.height, inf.width, 3), dtype=torch.uint8, device=dev)
            elif inf.channels == 1 and self.output != int(OutputColorspace.YCbCrPlanes):
                t = torch.empty((inf.height, inf.width), dtype=torch.uint8, device=dev)
            else:
                t = torch.empty((nb,), dtype=torch.uint8, device=dev)
            outs.append(t)
            ptrs.append(t.data_ptr())
            caps.append(t.numel())
        arr = (C.c_void_p * self.n)(*ptrs)
        carr = (C.c_size_t * self.n)(*caps)
        self._check(lib().pjg_batch_copy_outputs(self._h, arr, carr))
        ext = torch.cuda.ExternalStream(self.dec.stream(), device=dev)
        torch.cuda.current_stream(dev).wait_stream(ext)
        return outs

    def download(self, outs=None):
        """D2H into numpy buffers (allocated if not given); returns the list."""
        if outs is None:
            outs = [np.empty(max(1, int(inf.output_bytes)), np.uint8) for inf in self.infos]
        ptrs = (u8p * self.n)(*[o.ctypes.data_as(u8p) for o in outs])
        caps = (C.c_size_t * self.n)(*[o.size for o in outs])
        self._check(lib().pjg_batch_download(self._h, ptrs, caps))
        return outs

    def download_all(self, host_ptr: int, cap: int):
        """One D2H of the whole batch output into host memory at host_ptr."""
        self._check(lib().pjg_batch_download_all(self._h, C.c_void_p(host_ptr), cap))

    def download_all_async(self, host_ptr: int, cap: int):
        """Enqueue the batch output D2H on this context's stream (no wait)."""
        self._check(lib().pjg_batch_download_all_async(self._h, C.c_void_p(host_ptr), cap))

    def output_offset(self, i) -> int:
        return int(lib().pjg_batch_output_offset(self._h, i))

    def stage_times(self) -> StageTimings:
        ms = (C.c_double * 7)()
        self._check(lib().pjg_batch_stage_times(self._h, ms))
        return StageTimings(*[float(v) for v in ms])

    def sync_stats(self) -> dict:
        s = (C.c_uint64 * 8)()
        self._check(lib().pjg_batch_sync_stats(self._h, s))
        return {"intra_rounds_sum": int(s[0]), "intra_rounds_max": int(s[1]),
                "inter_hops": int(s[2]), "fixup_passes": int(s[3]),
                "k4_fp64_replayed_samples": int(s[4]), "k4_ac_units": int(s[5]),
                "compact_entries": int(s[6]), "compact": bool(s[7])}

    # ---- parity taps ----------------------------------------------------
    def coefficients(self, i, pre_dc_zigzag=True) -> np.ndarray:
        n = int(self.infos[i].data_units) * 64
        out = np.empty(max(n, 1), np.int16)
        self._check(lib().pjg_batch_dump_coefficients(self._h, i, 1 if pre_dc_zigzag else 0,
                                                      out.ctypes.data_as(C.c_void_p), out.size))
        return out[:n]

    def sync_states(self, i) -> np.ndarray:
        """(N, 5) uint64: p, trimmed n, c, z, divergent per subsequence."""
        n = C.c_size_t()
        self._check(lib().pjg_batch_dump_sync_states(self._h, i, None, 0, C.byref(n)))
        arr = (_SyncEntry * max(1, n.value))()
        self._check(lib().pjg_batch_dump_sync_states(self._h, i, arr, n.value, C.byref(n)))
        return np.array([[e.p, e.n, e.c, e.z, e.divergent] for e in arr[: n.value]],
                        np.uint64).reshape(-1, 5)

    def segment(self, i) -> bytes:
        n = C.c_size_t()
        self._check(lib().pjg_batch_dump_segment(self._h, i, None, 0, C.byref(n)))
        out = np.empty(max(1, n.value), np.uint8)
        self._check(lib().pjg_batch_dump_segment(self._h, i, out.ctypes.data_as(C.c_void_p),
                                                 out.size, C.byref(n)))
        return out[: n.value].tobytes()

    def close(self):
        if self._h:
            lib().pjg_batch_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------ drop-in API --
_default = threading.local()


def _decoder() -> Decoder:
    d = getattr(_default, "dec", None)
    if d is None:
        d = Decoder(int(os.environ.get("PJG_DEVICE", "0")))
        _default.dec = d
    return d


def _planes_from(buf: np.ndarray, inf: _Info) -> ImagePlanes:
    planes, off = [], 0
    for c in range(inf.num_components):
        w, h = inf.plane_width[c], inf.plane_height[c]
        planes.append(Plane(w, h, buf[off: off + w * h].reshape(h, w).copy()))
        off += w * h
    return ImagePlanes(inf.width, inf.height, inf.h_max, inf.v_max, planes)


def _success(b: Batch, i: int, buf: np.ndarray, output: int) -> DecodeSuccess:
    inf = b.infos[i]
    t = b.stage_times()
    if output == OutputColorspace.YCbCrPlanes:
        planes = _planes_from(buf, inf)
    else:  # RGB / gray are returned through the planes container's first plane
        ch = inf.channels
        pix = buf[: inf.width * inf.height * ch]
        planes = ImagePlanes(inf.width, inf.height, inf.h_max, inf.v_max,
                             [Plane(inf.width, inf.height,
                                    pix.reshape(inf.height, inf.width, ch) if ch == 3
                                    else pix.reshape(inf.height, inf.width))])
    return DecodeSuccess(planes, t, int(inf.compressed_bytes))


def decode_single(file_bytes, config: DecodeConfig | None = None) -> DecodeSuccess:
    """pjpeg::decode_single (pipeline.hpp:103-143) on the GPU: raises
    :class:`Error` with the reference's Errc on failure."""
    config = config or DecodeConfig()
    with _decoder().batch([file_bytes], config, OutputColorspace.YCbCrPlanes) as b:
        st = b.run()
        if st[0]:
            raise Error(int(st[0]), "decode_single")
        outs = b.download()
        return _success(b, 0, outs[0], OutputColorspace.YCbCrPlanes)


def decode_batch(files, config: DecodeConfig | None = None):
    """pjpeg::decode_batch (pipeline.hpp:147-163): per-file isolation; returns
    DecodeSuccess / DecodeFailure in input order."""
    config = config or DecodeConfig()
    if not files:
        return []
    with _decoder().batch(list(files), config, OutputColorspace.YCbCrPlanes) as b:
        st = b.run()
        outs = b.download()
        res = []
        for i in range(b.n):
            if st[i]:
                res.append(DecodeFailure(Errc(int(st[i]) - 1), _status_name(int(st[i]))))
            else:
                res.append(_success(b, i, outs[i], OutputColorspace.YCbCrPlanes))
        return res


def decode_to_tensors(files, device: int = 0, config: DecodeConfig | None = None,
                      output=OutputColorspace.RGBInterleaved, decoder: "Decoder | None" = None):
    """Decodes a batch straight into CUDA uint8 torch tensors on `device`
    (RGB: (H, W, 3)); per-file statuses (0 = ok, else Errc + 1) alongside.
    No host copy of any pixel."""
    own = decoder is None
    dec = decoder or Decoder(device)
    try:
        with dec.batch(files, config or DecodeConfig(), output) as b:
            st = b.run()
            return b.tensors(), st
    finally:
        if own:
            import torch
            torch.cuda.synchronize(dec.device)
            dec.close()


def decode_rgb(file_bytes, config: DecodeConfig | None = None) -> RgbImage:
    """decode_single + upsample_and_convert fused on the GPU (K4)."""
    config = config or DecodeConfig()
    with _decoder().batch([file_bytes], config, OutputColorspace.RGBInterleaved) as b:
        st = b.run()
        if st[0]:
            raise Error(int(st[0]), "decode_rgb")
        buf = b.download()[0]
        inf = b.infos[0]
        ch = inf.channels
        pix = buf[: inf.width * inf.height * ch]
        pix = pix.reshape(inf.height, inf.width, ch) if ch == 3 else pix.reshape(inf.height, inf.width)
        return RgbImage(inf.width, inf.height, pix.copy(), ch)


def upsample_and_convert(planes: ImagePlanes) -> RgbImage:
    """pjpeg::upsample_and_convert (pipeline.hpp:167-201) on the GPU (K5)."""
    n = len(planes.planes)
    W, H = planes.width, planes.height
    if n == 1:
        s = planes.planes[0].samples
        return RgbImage(W, H, np.ascontiguousarray(s[:H, :W]).copy(), 1)
    pw = (C.c_uint32 * 3)(*[p.width for p in planes.planes[:3]])
    ph = (C.c_uint32 * 3)(*[p.height for p in planes.planes[:3]])
    arrs = [np.ascontiguousarray(p.samples, np.uint8) for p in planes.planes[:3]]
    ptrs = (u8p * 3)(*[a.ctypes.data_as(u8p) for a in arrs])
    out = np.empty(W * H * 3, np.uint8)
    st = lib().pjg_upsample_and_convert(_decoder().handle, W, H, n, pw, ph, ptrs,
                                        out.ctypes.data_as(u8p))
    if st:
        raise Error(st, _decoder().last_error())
    return RgbImage(W, H, out.reshape(H, W, 3), 3)


def planes_checksum(planes: ImagePlanes) -> int:
    """pjpeg::planes_checksum (pipeline.hpp:204-215): FNV-1a over planes."""
    M = (1 << 64) - 1
    h = 1469598103934665603

    def mix(v):
        nonlocal h
        h ^= v
        h = (h * 1099511628211) & M

    mix(planes.width)
    mix(planes.height)
    for p in planes.planes:
        for s in np.asarray(p.samples, np.uint8).reshape(-1).tolist():
            mix(s)
    return h


def inspect(file_bytes, output=OutputColorspace.YCbCrPlanes) -> dict:
    """Header-only parse (no GPU needed): geometry + status."""
    a = np.frombuffer(file_bytes, np.uint8)
    inf = _Info()
    st = lib().pjg_inspect(a.ctypes.data_as(C.c_void_p), a.size, int(output), C.byref(inf))
    return {"status": int(st), "width": inf.width, "height": inf.height,
            "components": inf.num_components, "channels": inf.channels,
            "mcus_x": inf.mcus_x, "mcus_y": inf.mcus_y, "data_units": int(inf.data_units),
            "output_bytes": int(inf.output_bytes),
            "plane_dims": [(inf.plane_width[c], inf.plane_height[c])
                           for c in range(inf.num_components)]}


def decode_to_host_pipelined(decoders, blob, offsets, sizes, host_ptr: int, host_cap: int,
                             config: DecodeConfig | None = None, output=OutputColorspace.RGBInterleaved,
                             chunk: int = 512):
    """decode_batch into pinned host memory with copy/compute overlap.

    The batch (files laid out contiguously in ``blob``) is cut into chunks of
    ``chunk`` images that rotate over ``decoders`` (>= 2 contexts = 2 CUDA
    streams): chunk i's D2H runs while chunk i+1 is parsed on the host,
    uploaded and decoded.  Chunk outputs land back to back at ``host_ptr``.
    Returns (statuses, [(first_image, batch_output_offset_base, Batch)...] is
    not kept: returns statuses and per-chunk output byte offsets)."""
    config = config or DecodeConfig()
    n = len(sizes)
    live = [None] * len(decoders)
    statuses = np.zeros(n, np.int32)
    chunk_base = []
    base = 0
    pending = []

    def retire(slot):
        b, lo = live[slot]
        st = b.synchronize()
        statuses[lo: lo + len(st)] = st
        b.close()
        live[slot] = None

    for ci, lo in enumerate(range(0, n, chunk)):
        hi = min(n, lo + chunk)
        slot = ci % len(decoders)
        if live[slot] is not None:
            retire(slot)
        b = decoders[slot].batch((blob, offsets[lo:hi], sizes[lo:hi]), config, output)
        ob = b.output_bytes()
        if base + ob > host_cap:
            raise Error(int(Status_CAPACITY), "host buffer too small")
        b.upload()
        b.decode()
        b.download_all_async(host_ptr + base, host_cap - base)
        chunk_base.append(base)
        base += ob
        live[slot] = (b, lo)
    for slot in range(len(decoders)):
        if live[slot] is not None:
            retire(slot)
    return statuses, chunk_base, base


Status_CAPACITY = 102
