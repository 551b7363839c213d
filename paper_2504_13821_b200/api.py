"""Python mirror of the reference's public API for the TRMM/TRSM path.

Same names, argument meaning and error behaviour as the reference's C++
headers (paths relative to /root/reference/proj):

  flags.hpp       Side, Uplo, Trans, Diag, TriangularSpec, effective_op,
                  validate, parse_*, variant_string            (:10-77)
  matrix.hpp      MatrixBuffer, MatrixView, overlaps, split_half (:14-183)
  backend.hpp     GemmBlocking, Backend                         (:11-37)
  recursion.hpp   Threshold, DiagBlock, BHalf, GemmUpdate, RecursionSchema,
                  OpKind, schema_for, RecEvent, rec_trmm, rec_trsm (:11-86)
  base_kernels.hpp kDefaultTileLimit, trmm_base, trsm_base      (:9-30)
  gemm.hpp        gemm, scale                                   (:18-33)

Storage is a torch tensor (device memory for the in-place GPU path, host
memory for the staged path); every computation runs in librectri_cu.so on
the GPU -- there is no CPU compute path here.
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import torch

from . import _lib
from .errors import (
    BoundsError,
    ConfigError,
    ShapeError,
    SplitError,
    raise_for_status,
)

# ---------------------------------------------------------------------------
# flags.hpp


class Side(enum.IntEnum):
    Left = 0
    Right = 1


class Uplo(enum.IntEnum):
    Lower = 0
    Upper = 1


class Trans(enum.IntEnum):
    NoTrans = 0
    Trans = 1
    ConjTrans = 2


class Diag(enum.IntEnum):
    NonUnit = 0
    Unit = 1


class ElemKind(enum.IntEnum):
    F32 = 0
    F64 = 1


@dataclass
class TriangularSpec:
    side: Side = Side.Left
    uplo: Uplo = Uplo.Lower
    trans: Trans = Trans.NoTrans
    diag: Diag = Diag.NonUnit
    alpha: float = 1.0


def effective_op(trans, kind: ElemKind = ElemKind.F64) -> Trans:
    """ConjTrans reduces to Trans on real element kinds (flags.hpp:38-45)."""
    if isinstance(trans, TriangularSpec):
        trans = trans.trans
    return Trans.Trans if Trans(trans) == Trans.ConjTrans else Trans(trans)


def validate(spec: TriangularSpec) -> None:
    if not math.isfinite(spec.alpha):
        raise ConfigError("alpha must be finite")


_SIDE = {"left": Side.Left, "right": Side.Right}
_UPLO = {"lower": Uplo.Lower, "upper": Uplo.Upper}
_TRANS = {"n": Trans.NoTrans, "t": Trans.Trans, "c": Trans.ConjTrans}
_DIAG = {"unit": Diag.Unit, "nonunit": Diag.NonUnit}


def _parse(table, s: str, what: str, choices: str):
    if s not in table:
        raise ConfigError(f"unknown {what} '{s}' ({choices})")
    return table[s]


def parse_side(s: str) -> Side:
    return _parse(_SIDE, s, "side", "left|right")


def parse_uplo(s: str) -> Uplo:
    return _parse(_UPLO, s, "uplo", "lower|upper")


def parse_trans(s: str) -> Trans:
    return _parse(_TRANS, s, "trans", "n|t|c")


def parse_diag(s: str) -> Diag:
    return _parse(_DIAG, s, "diag", "unit|nonunit")


def to_string(x) -> str:
    if isinstance(x, Side):
        return "left" if x == Side.Left else "right"
    if isinstance(x, Uplo):
        return "lower" if x == Uplo.Lower else "upper"
    if isinstance(x, Trans):
        return {Trans.NoTrans: "n", Trans.Trans: "t"}.get(x, "c")
    if isinstance(x, Diag):
        return "nonunit" if x == Diag.NonUnit else "unit"
    if isinstance(x, OpKind):
        return "trmm" if x == OpKind.Trmm else "trsm"
    raise TypeError(type(x))


def variant_string(spec: TriangularSpec) -> str:
    """"left-lower-n-nonunit" (flags.cpp:30-40)."""
    return "-".join(to_string(v) for v in (Side(spec.side), Uplo(spec.uplo), Trans(spec.trans), Diag(spec.diag)))


# ---------------------------------------------------------------------------
# matrix.hpp

_DTYPES = {torch.float32: ElemKind.F32, torch.float64: ElemKind.F64}


class MatrixView:
    """Non-owning column-major window: element (r, c) lives at
    ``origin.flatten()[(col_offset + c) * origin_rows + row_offset + r]``;
    ``leading_dim`` is always the origin's row count (matrix.hpp:75-160)."""

    __slots__ = ("_origin", "_orows", "_ocols", "_r0", "_c0", "_rows", "_cols", "_const")

    def __init__(self, origin: torch.Tensor, origin_rows: int, origin_cols: int,
                 row_offset: int = 0, col_offset: int = 0,
                 rows: Optional[int] = None, cols: Optional[int] = None, const: bool = False):
        if origin.dtype not in _DTYPES:
            raise ConfigError(f"unsupported element type {origin.dtype}")
        if not origin.is_contiguous():
            raise ConfigError("origin tensor must be contiguous")
        if origin.numel() < origin_rows * origin_cols:
            raise ShapeError("origin tensor smaller than origin_rows * origin_cols")
        self._origin = origin
        self._orows, self._ocols = int(origin_rows), int(origin_cols)
        self._r0, self._c0 = int(row_offset), int(col_offset)
        self._rows = self._orows - self._r0 if rows is None else int(rows)
        self._cols = self._ocols - self._c0 if cols is None else int(cols)
        self._const = const

    # accessors (matrix.hpp:99-105)
    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def row_offset(self) -> int:
        return self._r0

    def col_offset(self) -> int:
        return self._c0

    def leading_dim(self) -> int:
        return self._orows

    def empty(self) -> bool:
        return self._rows == 0 or self._cols == 0

    def origin_id(self) -> int:
        return self._origin.data_ptr()

    @property
    def origin(self) -> torch.Tensor:
        return self._origin

    @property
    def dtype(self) -> torch.dtype:
        return self._origin.dtype

    @property
    def device(self) -> torch.device:
        return self._origin.device

    def as_const(self) -> "MatrixView":
        return MatrixView(self._origin, self._orows, self._ocols, self._r0, self._c0,
                          self._rows, self._cols, const=True)

    def subview(self, r0: int, c0: int, nr: int, nc: int) -> "MatrixView":
        """matrix.hpp:132-143"""
        if r0 < 0 or c0 < 0 or nr < 0 or nc < 0 or r0 + nr > self._rows or c0 + nc > self._cols:
            raise BoundsError(f"subview ({r0}, {c0}, {nr}, {nc}) escapes a {self._rows}x{self._cols} view")
        return MatrixView(self._origin, self._orows, self._ocols, self._r0 + r0, self._c0 + c0,
                          nr, nc, self._const)

    def tensor(self) -> torch.Tensor:
        """The window as a (rows, cols) strided torch view (no copy)."""
        flat = self._origin.reshape(-1)
        base = flat[: self._orows * self._ocols].view(self._ocols, self._orows)
        return base[self._c0: self._c0 + self._cols, self._r0: self._r0 + self._rows].t()

    def _c(self) -> _lib.View:
        return _lib.View(self._origin.data_ptr(), self._orows, self._ocols, self._r0, self._c0,
                         self._rows, self._cols)


class MatrixBuffer:
    """Owned column-major storage (matrix.hpp:18-70), on any torch device."""

    def __init__(self, rows: int, cols: int, dtype=torch.float64, device="cuda", fill: float = 0.0,
                 pin_memory: bool = False):
        if rows < 0 or cols < 0:
            raise ShapeError("negative matrix dimension")
        self._rows, self._cols = int(rows), int(cols)
        self.data = torch.full((max(cols, 0), max(rows, 0)), fill, dtype=dtype, device=device,
                               pin_memory=pin_memory and torch.device(device).type == "cpu")

    @classmethod
    def from_tensor(cls, t: torch.Tensor, device=None) -> "MatrixBuffer":
        """From a (rows, cols) tensor/array (copied into column-major storage)."""
        t = torch.as_tensor(t)
        out = cls.__new__(cls)
        out._rows, out._cols = t.shape
        out.data = t.t().contiguous().to(device if device is not None else t.device)
        return out

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def view(self) -> MatrixView:
        return MatrixView(self.data, self._rows, self._cols)

    def cview(self) -> MatrixView:
        return self.view().as_const()

    def tensor(self) -> torch.Tensor:
        return self.data.t()

    def numpy(self):
        return self.data.t().cpu().numpy()

    def clone(self) -> "MatrixBuffer":
        out = MatrixBuffer.__new__(MatrixBuffer)
        out._rows, out._cols = self._rows, self._cols
        out.data = self.data.clone()
        return out


def overlaps(a: MatrixView, b: MatrixView) -> bool:
    """matrix.hpp:168-177"""
    if a.origin_id() != b.origin_id():
        return False
    if a.empty() or b.empty():
        return False
    rows_meet = a.row_offset() < b.row_offset() + b.rows() and b.row_offset() < a.row_offset() + a.rows()
    cols_meet = a.col_offset() < b.col_offset() + b.cols() and b.col_offset() < a.col_offset() + a.cols()
    return rows_meet and cols_meet


def split_half(n: int) -> int:
    """matrix.hpp:180-183"""
    if n < 2:
        raise SplitError(f"cannot split dimension {n}")
    return n // 2


# ---------------------------------------------------------------------------
# backend.hpp


@dataclass
class GemmBlocking:
    mc: int = 64
    kc: int = 64
    nc: int = 64


ASYNC = 1
NO_GRAPH = 2
TF32X3 = 4  # fp32 GEMM updates as 3xTF32 on tcgen05 (opt-in variant, own tolerance)


@dataclass
class Backend:
    """backend.hpp:20-29 plus the device, stream and launch flags of the CUDA
    library.  ``parallel_width`` is validated (>= 1) like the reference and is
    otherwise advisory: parallelism is the CUDA grid, and results do not
    depend on it (the reference's par == seq guarantee)."""

    name: str = "cuda"
    parallel_width: int = 1
    blocking: GemmBlocking = field(default_factory=GemmBlocking)
    device: int = -1
    stream: object = None  # torch.cuda.Stream, raw handle (int) or None = torch's current stream
    flags: int = 0

    @staticmethod
    def seq() -> "Backend":
        return Backend(name="seq")

    @staticmethod
    def par(width: int = 0) -> "Backend":
        import os

        return Backend(name="par", parallel_width=width if width > 0 else max(1, os.cpu_count() or 1))

    @staticmethod
    def cuda(device: int = -1, stream=None, flags: int = 0) -> "Backend":
        return Backend(name="cuda", device=device, stream=stream, flags=flags)

    def _c(self, tensor_device: Optional[torch.device] = None) -> _lib.BackendC:
        stream = self.stream
        dev = self.device
        if dev < 0 and tensor_device is not None and tensor_device.type == "cuda":
            dev = tensor_device.index if tensor_device.index is not None else torch.cuda.current_device()
        if stream is None:
            handle = _current_stream_handle(dev)
        elif isinstance(stream, int):
            handle = stream
        else:
            handle = stream.cuda_stream
        return _lib.BackendC(self.parallel_width, dev, handle or None, self.flags,
                             self.blocking.mc, self.blocking.kc, self.blocking.nc)


# ---------------------------------------------------------------------------
# recursion.hpp

kDefaultTileLimit = 256


@dataclass
class Threshold:
    value: int = kDefaultTileLimit


class DiagBlock(enum.IntEnum):
    A11 = 0
    A22 = 1


class BHalf(enum.IntEnum):
    B1 = 0
    B2 = 1


@dataclass
class GemmUpdate:
    off_trans: Trans = Trans.NoTrans
    off_on_left: bool = True
    read_half: BHalf = BHalf.B1
    write_half: BHalf = BHalf.B2
    sign: float = 1.0
    carries_alpha: bool = False


@dataclass
class RecursionSchema:
    first_block: DiagBlock
    update: GemmUpdate
    second_block: DiagBlock


class OpKind(enum.IntEnum):
    Trmm = 0
    Trsm = 1


def parse_op_kind(s: str) -> OpKind:
    if s == "trmm":
        return OpKind.Trmm
    if s == "trsm":
        return OpKind.Trsm
    raise ConfigError(f"unknown op '{s}' (trmm|trsm)")


class RecEvent(enum.IntEnum):
    Gemm = 0
    BaseTrmm = 1
    BaseTrsm = 2


EventSink = Callable[[RecEvent, int, int], None]


def _current_stream_handle(dev: int) -> int:
    """torch's current stream on `dev` as a raw handle (the raw accessor skips
    building a torch.cuda.Stream object: ~0.3 us instead of ~3 us per call)."""
    if not torch.cuda.is_available():
        return 0
    d = dev if dev >= 0 else torch.cuda.current_device()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    return raw(d) if raw is not None else torch.cuda.current_stream(d).cuda_stream


_NULL_SINK = None


def _spec_c(spec: TriangularSpec) -> _lib.Spec:
    return _lib.Spec(int(spec.side), int(spec.uplo), int(spec.trans), int(spec.diag), float(spec.alpha))


def schema_for(op: OpKind, spec: TriangularSpec) -> RecursionSchema:
    """recursion.cpp:18-46, evaluated by the library's own table."""
    out = (ctypes.c_double * 8)()
    lib = _lib.load()
    st = lib.rectri_cu_schema_for(int(op), ctypes.byref(_spec_c(spec)), out)
    raise_for_status(st, _lib.last_error())
    upd = GemmUpdate(Trans(int(out[1])), bool(out[2]), BHalf(int(out[3])), BHalf(int(out[4])),
                     float(out[5]), bool(out[6]))
    return RecursionSchema(DiagBlock(int(out[0])), upd, DiagBlock(int(out[7])))


def _suffix(a: MatrixView, b: MatrixView) -> str:
    if a.dtype != b.dtype:
        raise ConfigError("A and B must have the same element type")
    return "f64" if a.dtype == torch.float64 else "f32"


def _sink_c(sink: Optional[EventSink]):
    global _NULL_SINK
    if sink is None:
        if _NULL_SINK is None:
            _NULL_SINK = _lib.EVENT_FN()
        return _NULL_SINK, None
    errors = []

    def tramp(_user, ev, n, m):
        try:
            sink(RecEvent(ev), int(n), int(m))
        except BaseException as e:  # re-raised after the call returns
            errors.append(e)

    return _lib.EVENT_FN(tramp), errors


def _device_of(*views: MatrixView) -> Optional[torch.device]:
    for v in views:
        if v.device.type == "cuda":
            return v.device
    return None


def _rec(op: OpKind, spec: TriangularSpec, A: MatrixView, B: MatrixView, threshold, backend, sink):
    lib = _lib.load()
    thr = threshold.value if isinstance(threshold, Threshold) else int(threshold)
    backend = backend if backend is not None else Backend.cuda()
    fn_c, errors = _sink_c(sink)
    sfx = _suffix(A, B)
    be = backend._c(_device_of(A, B))
    if op == OpKind.Trmm:
        st = getattr(lib, f"rectri_cu_rec_trmm_{sfx}")(ctypes.byref(_spec_c(spec)), A._c(), B._c(), thr,
                                                       ctypes.byref(be), fn_c, None)
        row = -1
    else:
        r = ctypes.c_int64(-1)
        st = getattr(lib, f"rectri_cu_rec_trsm_{sfx}")(ctypes.byref(_spec_c(spec)), A._c(), B._c(), thr,
                                                       ctypes.byref(be), fn_c, None, ctypes.byref(r))
        row = r.value
    if errors:
        raise errors[0]
    raise_for_status(st, _lib.last_error() if st else "", row)


def rec_trmm(spec: TriangularSpec, A: MatrixView, B: MatrixView, threshold=Threshold(),
             backend: Optional[Backend] = None, sink: Optional[EventSink] = None) -> None:
    """B <- alpha * op(A) * B (Left) or alpha * B * op(A) (Right), in place
    (recursion.hpp:66-75)."""
    _rec(OpKind.Trmm, spec, A, B, threshold, backend, sink)


def rec_trsm(spec: TriangularSpec, A: MatrixView, B: MatrixView, threshold=Threshold(),
             backend: Optional[Backend] = None, sink: Optional[EventSink] = None) -> None:
    """Solves op(A) X = alpha B (Left) or X op(A) = alpha B (Right), X stored in
    B (recursion.hpp:77-86).  Raises SingularityError with the global row of
    the first zero pivot met in leaf order."""
    _rec(OpKind.Trsm, spec, A, B, threshold, backend, sink)


def trmm_base(spec: TriangularSpec, A: MatrixView, B: MatrixView, tile_limit: int = kDefaultTileLimit,
              backend: Optional[Backend] = None) -> None:
    """base_kernels.hpp:15-19"""
    lib = _lib.load()
    backend = backend if backend is not None else Backend.cuda()
    st = getattr(lib, f"rectri_cu_trmm_base_{_suffix(A, B)}")(
        ctypes.byref(_spec_c(spec)), A._c(), B._c(), int(tile_limit), ctypes.byref(backend._c(_device_of(A, B))))
    raise_for_status(st, _lib.last_error() if st else "")


def trsm_base(spec: TriangularSpec, A: MatrixView, B: MatrixView, tile_limit: int = kDefaultTileLimit,
              backend: Optional[Backend] = None) -> None:
    """base_kernels.hpp:21-30 (zero pivots raise before B is touched; the
    index is tile-local)."""
    lib = _lib.load()
    backend = backend if backend is not None else Backend.cuda()
    r = ctypes.c_int64(-1)
    st = getattr(lib, f"rectri_cu_trsm_base_{_suffix(A, B)}")(
        ctypes.byref(_spec_c(spec)), A._c(), B._c(), int(tile_limit),
        ctypes.byref(backend._c(_device_of(A, B))), ctypes.byref(r))
    raise_for_status(st, _lib.last_error() if st else "", r.value)


def gemm(alpha: float, trans_a: Trans, A: MatrixView, trans_b: Trans, B: MatrixView, beta: float,
         C: MatrixView, backend: Optional[Backend] = None) -> None:
    """C <- alpha op(A) op(B) + beta C (gemm.hpp:18-21)."""
    lib = _lib.load()
    backend = backend if backend is not None else Backend.cuda()
    sfx = _suffix(A, C)
    _suffix(B, C)
    st = getattr(lib, f"rectri_cu_gemm_{sfx}")(float(alpha), int(trans_a), A._c(), int(trans_b), B._c(),
                                               float(beta), C._c(), ctypes.byref(backend._c(_device_of(A, B, C))))
    raise_for_status(st, _lib.last_error() if st else "")


def scale(alpha: float, B: MatrixView, backend: Optional[Backend] = None) -> None:
    """B <- alpha B (gemm.hpp:30-33)."""
    lib = _lib.load()
    backend = backend if backend is not None else Backend.cuda()
    sfx = "f64" if B.dtype == torch.float64 else "f32"
    st = getattr(lib, f"rectri_cu_scale_{sfx}")(float(alpha), B._c(), ctypes.byref(backend._c(_device_of(B))))
    raise_for_status(st, _lib.last_error() if st else "")


def sync(stream=None) -> None:
    """Completes RECTRI_CU_ASYNC calls on `stream` and raises deferred
    singularity errors."""
    lib = _lib.load()
    handle = stream if isinstance(stream, int) else (
        stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream)
    r = ctypes.c_int64(-1)
    st = lib.rectri_cu_sync(handle or None, ctypes.byref(r))
    raise_for_status(st, _lib.last_error() if st else "", r.value)


def launch_count() -> int:
    return int(_lib.load().rectri_cu_launch_count())


def clear_graph_cache() -> None:
    _lib.load().rectri_cu_clear_graph_cache()


def release_staging() -> None:
    """Frees the host-operand path's device staging buffers."""
    _lib.load().rectri_cu_release_staging()


def device_bytes_held() -> int:
    """Device bytes held across calls (cached graphs' scratch + staging)."""
    return int(_lib.load().rectri_cu_device_bytes_held())


# ---------------------------------------------------------------------------
# Utilities (not reference entry points): device-side synthetic inputs, peak
# probe and per-kernel-class profiling.


def fill_uniform(B: MatrixView, col0: int = 0, global_rows: Optional[int] = None, seed: int = 42,
                 backend: Optional[Backend] = None) -> None:
    """Uniform [-1, 1) keyed by the global element index (col0 + c) *
    global_rows + r: shards generated anywhere reproduce the unsharded matrix."""
    lib = _lib.load()
    backend = backend if backend is not None else Backend.cuda()
    st = lib.rectri_cu_fill_uniform(1 if B.dtype == torch.float64 else 0, B._c(), int(col0),
                                    int(global_rows if global_rows is not None else B.rows()), int(seed),
                                    ctypes.byref(backend._c(_device_of(B))))
    raise_for_status(st, _lib.last_error() if st else "")


def make_dominant(A: MatrixView, uplo: Uplo = Uplo.Lower, backend: Optional[Backend] = None) -> None:
    """diag := stored off-diagonal |row sum| + 1 (src/bench.cpp:40-51), on the device."""
    lib = _lib.load()
    backend = backend if backend is not None else Backend.cuda()
    st = lib.rectri_cu_make_dominant(1 if A.dtype == torch.float64 else 0, A._c(), int(uplo),
                                     ctypes.byref(backend._c(_device_of(A))))
    raise_for_status(st, _lib.last_error() if st else "")


def debug_ring_check(reset: bool = True) -> int:
    """Mismatches the default fp64 leaf's ring checker counted
    (RECTRI_CU_RING_CHECK=1 at launch / capture; =2 plants a slot mix-up);
    synchronises the device.  The first call allocates the counter: call it
    once before the checked launches."""
    return int(_lib.load().rectri_cu_debug_ring_check(1 if reset else 0))


def probe_peak(kind: str = "f64") -> float:
    """Measured issue-rate peak in TFLOP/s: 'f64' = DMMA.8x8x4, 'f32' = FFMA."""
    return float(_lib.load().rectri_cu_probe_peak(0 if kind == "f64" else 1))


PROFILE_KINDS = ("gemm", "leaf", "scale", "scan")


def profile_enable(on: bool = True) -> None:
    _lib.load().rectri_cu_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kind: {"ms", "launches", "flops"}} since the last read."""
    ms = (ctypes.c_double * 4)()
    la = (ctypes.c_int64 * 4)()
    fl = (ctypes.c_double * 4)()
    st = _lib.load().rectri_cu_profile_read(ms, la, fl)
    raise_for_status(st, _lib.last_error() if st else "")
    return {k: {"ms": ms[i], "launches": int(la[i]), "flops": fl[i]} for i, k in enumerate(PROFILE_KINDS)}
