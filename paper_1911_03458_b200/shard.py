"""Multi-GPU sharding of a workload along its leading batch / frame-pair axis.

The MERIT outputs of different images (conv, max-pool) or frame pairs (motion
estimation) are independent ranged inner products, so a workload with a
leading p-axis that maps 1:1 onto a leading source axis of every view that
uses it shards with no exchange at all: rank r gets a
contiguous slice of that axis, runs the unchanged device plan on it, and the
output slices concatenate.  Views that do not use the batch component
(weights) are replicated.  No collective is on the data path.
"""
from __future__ import annotations

import copy
from typing import Tuple

import numpy as np

from .merit import Error, ErrorCode, Workload


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced split: [start, stop) of `total` items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise Error(ErrorCode.InvalidArgument, "bad rank/world")
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def _batch_axis_of(view, comp: int):
    """Source axis fed only by component `comp` with stride 1, or None if the
    view does not use `comp`."""
    axes = [t.axis for t in view.terms if t.component == comp]
    if not axes:
        return None
    ax = axes[0]
    ts = [t for t in view.terms if t.axis == ax]
    if len(axes) != 1 or len(ts) != 1 or ts[0].stride != 1 or ts[0].offset != 0:
        raise Error(ErrorCode.BadParams, "leading p-axis is not a plain batch axis")
    return ax


def shard_workload(w: Workload, world: int, rank: int) -> Tuple[Workload, Tuple[int, int]]:
    """Slice p-axis 0 of `w` for `rank`; returns (shard, (start, stop))."""
    total = w.view_a.p_shape[0]
    start, stop = shard_range(total, world, rank)
    s = copy.copy(w)
    s.view_a = copy.deepcopy(w.view_a)
    s.view_b = copy.deepcopy(w.view_b)
    for attr_v, attr_s in (("view_a", "src_a"), ("view_b", "src_b")):
        v = getattr(s, attr_v)
        v.p_shape[0] = stop - start
        ax = _batch_axis_of(v, 0)
        src = getattr(w, attr_s)
        if ax is None:
            continue  # replicated operand (e.g. weights)
        if ax != 0:
            raise Error(ErrorCode.BadParams, "batch axis must be the leading source axis")
        if v.source_shape[0] != total:
            raise Error(ErrorCode.BadParams, "batch extent differs between p and source")
        v.source_shape[0] = stop - start
        if src is not None:
            setattr(s, attr_s, np.ascontiguousarray(src[start:stop]))
    return s, (start, stop)


def _axis_footprint(view, axis: int, kshape, comp0_range) -> Tuple[int, int]:
    """Eq. 6 extent (view.hpp:121-149) of source axis `axis` over the index
    box kshape with component 0 restricted to comp0_range: [lo, hi]."""
    lo = hi = 0
    for t in view.terms:
        if t.axis != axis:
            continue
        if t.component == 0:
            a, b = comp0_range[0] * t.stride, (comp0_range[1] - 1) * t.stride
        else:
            a, b = 0, (kshape[t.component] - 1) * t.stride
        lo += min(a, b) + t.offset
        hi += max(a, b) + t.offset
    return lo, hi


def shard_band(w: Workload, world: int, rank: int) -> Tuple[Workload, Tuple[int, int]]:
    """Band split of a single-image workload along p-axis 0 (e.g. the block
    rows of one motion-estimation frame pair): rank r gets
    a contiguous range of p-axis 0 and, of every source that the component
    feeds through source axis 0, only the rows its band reads — the Eq. 6
    footprint of the band (footprint_box, view.hpp:121-149), i.e. its rows
    plus the search-window halo — sliced at load time.  The view's axis-0
    offset is shifted by the slice start, so every gather reads the same
    value as in the unsplit workload (rows outside the original source stay
    outside the slice: ZERO_PAD / CLAMP / REJECT behave identically).  No
    exchange between ranks.

    The shard records where its source slices start in the original sources
    (``shard.row_origin = (rows of src_a, rows of src_b)``): outputs are
    identical, but anything expressed in source coordinates — e.g. the
    argmin records' motion vector, ref row - cur row — is relative to the
    slices and shifts by row_origin[ref] - row_origin[cur]."""
    total = w.view_a.p_shape[0]
    start, stop = shard_range(total, world, rank)
    kshape = list(w.view_a.p_shape) + list(w.view_a.a_shape)
    s = copy.copy(w)
    origin = [0, 0]
    s.view_a = copy.deepcopy(w.view_a)
    s.view_b = copy.deepcopy(w.view_b)
    for side, (attr_v, attr_s) in enumerate((("view_a", "src_a"), ("view_b", "src_b"))):
        v = getattr(s, attr_v)
        v.p_shape[0] = stop - start
        uses0 = [t for t in v.terms if t.component == 0]
        if not uses0:
            continue  # replicated operand
        if any(t.axis != 0 for t in uses0):
            raise Error(ErrorCode.BadParams, "band component must feed source axis 0 only")
        if stop <= start:
            continue
        lo, hi = _axis_footprint(getattr(w, attr_v), 0, kshape, (start, stop))
        rows = v.source_shape[0]
        r0, r1 = max(0, lo), min(rows - 1, hi)
        if r1 < r0:  # the band reads nothing inside the source: keep one row
            r0 = r1 = min(max(0, lo), rows - 1)
        v.source_shape[0] = r1 - r0 + 1
        # component 0 now counts from 0: fold start*stride - r0 into one term
        t0 = next(t for t in v.terms if t.component == 0)
        t0.offset += start * t0.stride - r0
        origin[side] = r0
        src = getattr(w, attr_s)
        if src is not None:
            setattr(s, attr_s, np.ascontiguousarray(src[r0:r1 + 1]))
    s.row_origin = tuple(origin)
    return s, (start, stop)
