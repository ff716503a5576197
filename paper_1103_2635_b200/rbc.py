"""Random ball cover index: sampling, builds, parameter formulas (reference rbc.py).

Both builds run on the GPU through the C-ABI and return the reference
dataclasses (``RbcExactIndex`` / ``RbcOneShotIndex``) with host numpy fields,
plus a device-resident index handle (``index._dev``) that the searches use
without re-uploading anything.  An index constructed by hand (e.g. from saved
arrays) is uploaded on first search.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .dataset import DataMatrix, FormatError
from .metric import MetricSpec

BERNOULLI = "bernoulli"
FIXED_COUNT = "fixed-count"
_MODES = (BERNOULLI, FIXED_COUNT)


@dataclass(frozen=True)
class RepSet:
    """The sampled representative ids (sorted ascending) and how they were drawn (rbc.py:44-54)."""

    rep_ids: np.ndarray
    sampling_mode: str
    seed: int

    @property
    def size(self) -> int:
        return len(self.rep_ids)


def _pcg64_words(seed: int):
    """128-bit PCG64 state/increment of numpy's default_rng(seed) (SeedSequence seeding, host)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return s >> 64, s & m, inc >> 64, inc & m


def _bernoulli_draw(n: int, p: float, seed: int) -> np.ndarray:
    """rbc.py:57-59 on the device: ids i with default_rng(seed).random(n)[i] < p."""
    t = _lib.require_cuda()
    out = _lib.empty((n,), t.int64)
    count = ctypes.c_int64(0)
    _lib.check(_lib.lib.rbc_bernoulli_draw(n, float(p), *_pcg64_words(seed), _lib.ptr(out), ctypes.byref(count),
                                           _lib.stream_ptr()), "bernoulli draw")
    return _lib.to_host(out[: count.value])


def sample_representatives(n: int, n_r: int, seed: int, mode: str = BERNOULLI) -> RepSet:
    """Draw the representative set (rbc.py:62-84)."""
    if not 1 <= n_r <= n:
        raise ValueError(f"n_r must be in [1, {n}], got {n_r}")
    if mode not in _MODES:
        raise ValueError(f"unknown sampling mode {mode!r}; expected one of {_MODES}")
    if seed < 0:
        raise ValueError("seed must be non-negative")
    if mode == BERNOULLI:
        ids = _bernoulli_draw(n, n_r / n, seed)
        if ids.size == 0:
            ids = _bernoulli_draw(n, n_r / n, seed + 1)
        if ids.size == 0:
            raise ValueError(f"bernoulli sampling produced an empty set twice (n={n}, n_r={n_r})")
    else:
        # O(n_r) host draw without replacement, identical to the reference's generator call
        rng = np.random.default_rng(seed)
        ids = np.sort(rng.choice(n, size=n_r, replace=False))
    return RepSet(np.asarray(ids, dtype=np.int64), mode, seed)


class DeviceIndex:
    """Owner of an rbc_index* handle (device-resident index)."""

    def __init__(self, handle: ctypes.c_void_p, device: int):
        self.handle = handle
        self.device = device

    @property
    def nbytes(self) -> int:
        return int(_lib.lib.rbc_index_device_bytes(self.handle))

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h is not None and h.value:
            try:
                _lib.lib.rbc_index_destroy(h)
            except Exception:  # interpreter shutdown
                pass


@dataclass
class RbcExactIndex:
    """Disjoint ownership partition for exact search (rbc.py:87-115)."""

    data: DataMatrix
    metric: MetricSpec
    reps: RepSet
    list_ids: list[np.ndarray]
    list_dists: list[np.ndarray]
    radii: np.ndarray

    @property
    def rep_points(self) -> np.ndarray:
        return np.ascontiguousarray(self.data.values[self.reps.rep_ids])

    def owner_positions(self) -> np.ndarray:
        owner = np.empty(self.data.n, dtype=np.int64)
        for pos, ids in enumerate(self.list_ids):
            owner[ids] = pos
        return owner

    def flat_lists(self):
        """(list_ids, offsets, list_dists) as flat CSR arrays."""
        lengths = np.array([len(a) for a in self.list_ids], np.int64)
        offsets = np.zeros(len(lengths) + 1, np.int64)
        np.cumsum(lengths, out=offsets[1:])
        ids = np.concatenate(self.list_ids).astype(np.int64) if len(self.list_ids) else np.empty(0, np.int64)
        dists = np.concatenate(self.list_dists).astype(np.float32) if len(self.list_dists) else np.empty(0, np.float32)
        return ids, offsets, dists


@dataclass
class RbcOneShotIndex:
    """Overlapping fixed-size ownership lists for one-shot search (rbc.py:118-137)."""

    data: DataMatrix
    metric: MetricSpec
    reps: RepSet
    list_ids: np.ndarray
    s: int
    radii: np.ndarray

    @property
    def rep_points(self) -> np.ndarray:
        return np.ascontiguousarray(self.data.values[self.reps.rep_ids])


def _resolve_reps(n: int, n_r: int, seed: int, mode: str, rep_ids) -> RepSet:
    if rep_ids is not None:
        ids = np.sort(np.asarray(rep_ids, dtype=np.int64))
        return RepSet(ids, mode, seed)
    return sample_representatives(n, n_r, seed, mode)


def _split(flat: np.ndarray, offsets: np.ndarray) -> list[np.ndarray]:
    # independent arrays per list, as the reference's np.split(...) copies (rbc.py:170-176)
    return [flat[offsets[p]: offsets[p + 1]].copy() for p in range(len(offsets) - 1)]


_INDEX_FIELDS = ("data", "metric", "reps", "list_ids", "list_dists", "radii", "s")


def _fingerprint(index):
    """Identity of the index's fields: the device copy is reused only while none of them has
    been reassigned (the arrays themselves are treated as immutable once built, like the
    reference's read-only DataMatrix)."""
    fp = []
    for f in _INDEX_FIELDS:
        v = getattr(index, f, None)
        fp.append(v if isinstance(v, int) else id(v))
    lists = getattr(index, "list_ids", None)
    fp.append(len(lists) if isinstance(lists, list) else None)
    return tuple(fp)


def _attach(index, dev):
    index._dev = dev
    index._dev_fp = _fingerprint(index)


def _create_exact_device(x_dev, n, spec, rep_dev, nr, ids_dev, off_dev, ld_dev, radii_dev, owned=None):
    handle = ctypes.c_void_p()
    if owned is None:
        rc = _lib.lib.rbc_index_exact_create(_lib.ptr(x_dev), n, spec.dim, spec.code, _lib.ptr(rep_dev), nr,
                                             _lib.ptr(ids_dev), _lib.ptr(off_dev), _lib.ptr(ld_dev),
                                             _lib.ptr(radii_dev), ctypes.byref(handle), _lib.stream_ptr())
    else:
        mask = np.ascontiguousarray(owned, dtype=np.uint8)
        rc = _lib.lib.rbc_index_exact_create_shard(_lib.ptr(x_dev), n, spec.dim, spec.code, _lib.ptr(rep_dev), nr,
                                                   _lib.ptr(ids_dev), _lib.ptr(off_dev), _lib.ptr(ld_dev),
                                                   _lib.ptr(radii_dev), mask.ctypes.data_as(ctypes.c_void_p),
                                                   ctypes.byref(handle), _lib.stream_ptr())
    _lib.check(rc, "index create")
    return DeviceIndex(handle, _lib.torch().cuda.current_device())


def build_exact(
    data: DataMatrix,
    n_r: int,
    spec: MetricSpec,
    seed: int,
    mode: str = BERNOULLI,
    rep_ids=None,
    workers: int | None = None,
) -> RbcExactIndex:
    """Build the exact-search index on the GPU (rbc.py:147-180)."""
    t = _lib.require_cuda()
    reps = _resolve_reps(data.n, n_r, seed, mode, rep_ids)
    if data.d != spec.dim:
        raise ValueError(f"dimension mismatch: data d={data.d}, metric dim={spec.dim}")
    n, nr = data.n, reps.size
    x_dev = _lib.to_device(data.values)
    rep_dev = _lib.to_device(reps.rep_ids)
    ids_dev = _lib.empty((n,), t.int64)
    off_dev = _lib.empty((nr + 1,), t.int64)
    ld_dev = _lib.empty((n,), t.float32)
    radii_dev = _lib.empty((nr,), t.float32)
    _lib.check(_lib.lib.rbc_build_exact(_lib.ptr(x_dev), n, spec.dim, spec.code, _lib.ptr(rep_dev), nr,
                                        _lib.ptr(ids_dev), _lib.ptr(off_dev), _lib.ptr(ld_dev), _lib.ptr(radii_dev),
                                        _lib.stream_ptr()), "build_exact")
    dev = _create_exact_device(x_dev, n, spec, rep_dev, nr, ids_dev, off_dev, ld_dev, radii_dev)
    flat_ids, offsets, flat_d = _lib.to_host(ids_dev), _lib.to_host(off_dev), _lib.to_host(ld_dev)
    index = RbcExactIndex(data, spec, reps, _split(flat_ids, offsets), _split(flat_d, offsets),
                          _lib.to_host(radii_dev))
    _attach(index, dev)
    return index


def build_one_shot(
    data: DataMatrix,
    n_r: int,
    s: int,
    spec: MetricSpec,
    seed: int,
    mode: str = BERNOULLI,
    rep_ids=None,
    workers: int | None = None,
) -> RbcOneShotIndex:
    """Build the one-shot index on the GPU (rbc.py:183-200)."""
    if not 1 <= s <= data.n:
        raise ValueError(f"s must be in [1, {data.n}], got {s}")
    t = _lib.require_cuda()
    reps = _resolve_reps(data.n, n_r, seed, mode, rep_ids)
    if data.d != spec.dim:
        raise ValueError(f"dimension mismatch: data d={data.d}, metric dim={spec.dim}")
    n, nr = data.n, reps.size
    x_dev = _lib.to_device(data.values)
    rep_dev = _lib.to_device(reps.rep_ids)
    lists_dev = _lib.empty((nr, s), t.int64)
    radii_dev = _lib.empty((nr,), t.float32)
    _lib.check(_lib.lib.rbc_build_one_shot(_lib.ptr(x_dev), n, spec.dim, spec.code, _lib.ptr(rep_dev), nr, s,
                                           _lib.ptr(lists_dev), _lib.ptr(radii_dev), _lib.stream_ptr()),
               "build_one_shot")
    handle = ctypes.c_void_p()
    _lib.check(_lib.lib.rbc_index_one_shot_create(_lib.ptr(x_dev), n, spec.dim, spec.code, _lib.ptr(rep_dev), nr,
                                                  _lib.ptr(lists_dev), s, _lib.ptr(radii_dev), ctypes.byref(handle),
                                                  _lib.stream_ptr()), "one-shot index")
    index = RbcOneShotIndex(data, spec, reps, _lib.to_host(lists_dev), s, _lib.to_host(radii_dev))
    _attach(index, DeviceIndex(handle, t.cuda.current_device()))
    return index


def device_index(index) -> DeviceIndex:
    """The index's device handle, uploading a hand-made / loaded index on first use."""
    t = _lib.require_cuda()
    dev = getattr(index, "_dev", None)
    if (dev is not None and dev.handle is not None and dev.device == t.cuda.current_device()
            and getattr(index, "_dev_fp", None) == _fingerprint(index)):
        return dev
    spec = index.metric
    x_dev = _lib.to_device(index.data.values)
    rep_dev = _lib.to_device(index.reps.rep_ids)
    radii_dev = _lib.to_device(np.asarray(index.radii, np.float32))
    if isinstance(index, RbcExactIndex):
        ids, offsets, dists = index.flat_lists()
        dev = _create_exact_device(x_dev, index.data.n, spec, rep_dev, index.reps.size, _lib.to_device(ids),
                                   _lib.to_device(offsets), _lib.to_device(dists), radii_dev)
    else:
        handle = ctypes.c_void_p()
        lists_dev = _lib.to_device(np.asarray(index.list_ids, np.int64))
        _lib.check(_lib.lib.rbc_index_one_shot_create(_lib.ptr(x_dev), index.data.n, spec.dim, spec.code,
                                                      _lib.ptr(rep_dev), index.reps.size, _lib.ptr(lists_dev),
                                                      index.s, _lib.ptr(radii_dev), ctypes.byref(handle),
                                                      _lib.stream_ptr()), "one-shot index")
        dev = DeviceIndex(handle, t.cuda.current_device())
    _attach(index, dev)
    return dev


def standard_params_exact(n: int, c: float) -> int:
    """Representative count ceil(c^1.5 sqrt(n)) (rbc.py:203-209)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if c < 1:
        raise ValueError(f"expansion-rate estimate must be >= 1, got {c}")
    return int(min(n, max(1, math.ceil(c**1.5 * math.sqrt(n)))))


def one_shot_params(n: int, c: float, delta: float) -> tuple[int, int]:
    """n_r = s = ceil(c sqrt(n) sqrt(ln(1/delta))) (rbc.py:212-225)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if c < 1:
        raise ValueError(f"expansion-rate estimate must be >= 1, got {c}")
    if not 0 < delta < 1:
        raise ValueError(f"delta must be in (0, 1), got {delta}")
    value = int(min(n, max(1, math.ceil(c * math.sqrt(n) * math.sqrt(math.log(1.0 / delta))))))
    return value, value


# ---- RBCI index files (rbc.py:13-18 format, :228-322 writer/reader) -------------------------------------------
#
# Layout, all little-endian 32-bit: b"RBCI", version, variant (0 exact / 1 one-shot), metric (0 l2 / 1 l1),
# sampling mode (0 bernoulli / 1 fixed-count), seed lo, seed hi, |R|, rep ids u32[|R|]; exact: list lengths
# u32[|R|], ids u32[n], dists f32[n]; one-shot: s, ids u32[|R|*s]; then radii f32[|R|], n, d, X f32[n*d].
# Files are byte-identical to the reference's, so an index built on the GPU can be loaded by the reference and
# vice versa (tests/test_index_files.py).

RBCI_MAGIC = b"RBCI"
RBCI_VERSION = 1


def save_index(index, path) -> None:
    """Write an exact or one-shot index with its embedded database (rbc.py:233-258)."""
    exact = isinstance(index, RbcExactIndex)
    seed = int(index.reps.seed)
    head = np.array([RBCI_VERSION, 0 if exact else 1, _lib.METRIC_CODE[index.metric.kind],
                     0 if index.reps.sampling_mode == BERNOULLI else 1, seed & 0xFFFFFFFF,
                     (seed >> 32) & 0xFFFFFFFF, index.reps.size], dtype="<u4")
    parts = [RBCI_MAGIC, head, np.asarray(index.reps.rep_ids).astype("<u4")]
    if exact:
        ids, offsets, dists = index.flat_lists()
        parts += [np.diff(offsets).astype("<u4"), ids.astype("<u4"), dists.astype("<f4")]
    else:
        parts += [np.array([index.s], "<u4"), np.asarray(index.list_ids).astype("<u4")]
    parts += [np.asarray(index.radii).astype("<f4"), np.array([index.data.n, index.data.d], "<u4"),
              np.asarray(index.data.values, dtype="<f4")]
    with open(path, "wb") as fh:
        for p in parts:
            fh.write(p if isinstance(p, bytes) else p.tobytes())


def load_index(path):
    """Read an RBCI file (rbc.py:284-322): bit-exact round trip; the device copy is uploaded on first search.

    ``FormatError`` on a bad magic, version or tag; ``OSError`` on a truncated file.
    """
    with open(path, "rb") as fh:
        buf = fh.read()
    at = 0

    def take(dtype, count):
        nonlocal at
        nbytes = np.dtype(dtype).itemsize * count
        if at + nbytes > len(buf):
            raise OSError(f"{path}: truncated index file")
        out = np.frombuffer(buf, dtype=dtype, count=count, offset=at)
        at += nbytes
        return out

    if bytes(take("S4", 1)[0]) != RBCI_MAGIC:
        raise FormatError(f"{path}: bad magic, expected {RBCI_MAGIC!r}")
    version = int(take("<u4", 1)[0])
    if version != RBCI_VERSION:
        raise FormatError(f"{path}: unsupported index version {version}")
    variant, metric_code, mode_code, seed_lo, seed_hi, nr = (int(v) for v in take("<u4", 6))
    if variant > 1 or metric_code > 1 or mode_code > 1:
        raise FormatError(f"{path}: invalid variant/metric/mode tags")
    reps = RepSet(take("<u4", nr).astype(np.int64), BERNOULLI if mode_code == 0 else FIXED_COUNT,
                  seed_lo | (seed_hi << 32))
    if variant == 0:
        lengths = take("<u4", nr).astype(np.int64)
        offsets = np.zeros(nr + 1, np.int64)
        np.cumsum(lengths, out=offsets[1:])
        total = int(offsets[-1])
        flat_ids = take("<u4", total).astype(np.int64)
        flat_d = take("<f4", total).astype(np.float32)
    else:
        s = int(take("<u4", 1)[0])
        lists = take("<u4", nr * s).astype(np.int64).reshape(nr, s)
    radii = take("<f4", nr).astype(np.float32)
    n, d = (int(v) for v in take("<u4", 2))
    data = DataMatrix(take("<f4", n * d).reshape(n, d).astype(np.float32))
    spec = MetricSpec("l2" if metric_code == 0 else "l1", d)
    if variant == 0:
        return RbcExactIndex(data, spec, reps, _split(flat_ids, offsets), _split(flat_d, offsets), radii)
    return RbcOneShotIndex(data, spec, reps, lists, s, radii)
