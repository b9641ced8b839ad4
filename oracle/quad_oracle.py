"""CPU oracle for the QUAD tick pipeline — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

This module restates, in columnar NumPy, the reference algorithm of the
`tickjoin` package (arXiv 1411.3212 desk-scale reimplementation) for the one
path this repository accelerates: the QUAD method's per-tick pipeline, and the
uniform-grid (UG) index that feeds the same join and decode.  It is
the checker that the CUDA path is compared against; only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import it.
The product (`paper_1411_3212_b200`) never imports it and fails loudly when
its CUDA library is missing.

Parity is pinned: `tests/test_oracle_golden.py` checks this restatement
against (a) the known-answer vectors of the reference's own tests
(`pkg/tests/test_quadtree.py`, `test_bitmap.py`, `test_decode.py`,
`test_morton.py`, `test_acceptance.py` C2/C3) and (b) fixtures produced by
running the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`, `*.json`).

Arithmetic follows the reference bit for bit: every float op is a separate
IEEE-754 binary64 NumPy/Python operation (no fused multiply-add), in the same
order as the cited lines.  Citations are `file:line` inside
`/root/reference/pkg/src/tickjoin/`.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

L_MAX = 12  # morton.py:20
WORD_BITS = 32  # bitmap.py:20


class OracleError(Exception):
    """Mirrors the reference exception classes by name (errors.py:4-45)."""

    def __init__(self, kind: str, msg: str = ""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# L0/L1: MBR, cell coordinates, Morton codes
# --------------------------------------------------------------------------

def mbr_of(xs: np.ndarray, ys: np.ndarray) -> tuple[float, float, float, float]:
    """Exact min/max bounding rectangle.  geometry.py:72-77."""
    if len(xs) == 0:
        raise OracleError("EmptyBatch", "no objects")
    return (float(xs.min()), float(ys.min()), float(xs.max()), float(ys.max()))


def cell_coords(xs, ys, mbr, level: int) -> tuple[np.ndarray, np.ndarray]:
    """Point -> level-`level` grid cell over `mbr`; upper edge clamps.

    morton.py:90-109: i = int(min((x - xa) * (2**level / width), 2**level - 1)),
    0 when width == 0; OutOfBounds when a point is outside the MBR.
    """
    xs = np.asarray(xs, dtype=np.float64)
    ys = np.asarray(ys, dtype=np.float64)
    xa, ya, xb, yb = mbr
    outside = (xs < xa) | (xs > xb) | (ys < ya) | (ys > yb)
    if np.any(outside):
        raise OracleError("OutOfBounds", "point outside the MBR")
    side = 1 << level
    width = xb - xa
    height = yb - ya
    if width > 0:
        scale = side / width  # Python float division, as morton.py:102
        i = np.minimum((xs - xa) * scale, side - 1).astype(np.int64)
    else:
        i = np.zeros(xs.shape, dtype=np.int64)
    if height > 0:
        scale = side / height
        j = np.minimum((ys - ya) * scale, side - 1).astype(np.int64)
    else:
        j = np.zeros(ys.shape, dtype=np.int64)
    return i, j


def _part1by1(v):
    """Move bit k of the low 16 bits to bit 2k (standard Morton spread)."""
    v = np.asarray(v, dtype=np.int64) & 0xFFFF
    out = np.zeros_like(v)
    for k in range(16):
        out |= ((v >> k) & 1) << (2 * k)
    return out


def _compact1by1(v):
    v = np.asarray(v, dtype=np.int64)
    out = np.zeros_like(v)
    for k in range(16):
        out |= ((v >> (2 * k)) & 1) << k
    return out


def morton(i, j):
    """x (column) bits on even positions, y (row) bits on odd.  morton.py:64-66."""
    return _part1by1(i) | (_part1by1(j) << 1)


def unmorton(z):
    """Inverse of `morton`.  morton.py:69-71."""
    z = np.asarray(z, dtype=np.int64)
    return _compact1by1(z), _compact1by1(z >> 1)


def pack(level, z, l_max: int):
    """Packed leaf id, level in the high bits.  quadtree.py:51-52."""
    return (np.asarray(level, dtype=np.int64) << (2 * l_max)) | np.asarray(z, dtype=np.int64)


# --------------------------------------------------------------------------
# L2: PR-quadtree (Alg. 1), z_map, object / query mapping
# --------------------------------------------------------------------------

@dataclass
class OracleIndex:
    mbr: tuple
    th_quad: int
    l_max: int
    l_deep: int
    leaves: np.ndarray  # packed ids ascending
    zmap: np.ndarray  # 4**l_deep packed ids
    trace: Optional[list] = None  # per level: list of (level, z, start, end, split)


def build_index(xs, ys, mbr, th_quad: int, l_max: int, record_trace: bool = False) -> OracleIndex:
    """Level-wise bulk construction over sorted l_max codes.  quadtree.py:74-139.

    A quadrant at level l is a child of a split quadrant (the root always
    splits, 103-106); it splits iff it holds more than th_quad objects and
    l < l_max (116), otherwise it is a leaf, empty children included (122).
    Counts are the sizes of code intervals in the sorted code vector (111-112).
    """
    if th_quad < 1:
        raise ValueError("th_quad must be >= 1")
    if not 1 <= l_max <= L_MAX:
        raise ValueError("l_max out of range")
    i, j = cell_coords(xs, ys, mbr, l_max)
    codes = np.sort(morton(i, j))
    n = len(codes)
    leaves = []
    trace = []
    parents = np.array([0], dtype=np.int64)  # z of split quadrants at level l-1
    p_start = np.array([0], dtype=np.int64)
    p_end = np.array([n], dtype=np.int64)
    l_deep = 1
    for level in range(1, l_max + 1):
        if len(parents) == 0:
            break
        shift = 2 * (l_max - level)
        child_z = (parents[:, None] * 4 + np.arange(4)[None, :]).reshape(-1)
        # interval of each child: codes whose level-`level` prefix equals child_z
        lo = np.searchsorted(codes, child_z << shift, side="left")
        hi = np.searchsorted(codes, (child_z + 1) << shift, side="left")
        cnt = hi - lo
        split = (cnt > th_quad) & (level < l_max)
        if record_trace:
            trace.append([(level, int(z), int(s), int(e), bool(sp))
                          for z, s, e, sp in zip(child_z, lo, hi, split)])
        leaves.append(pack(level, child_z[~split], l_max))
        parents = child_z[split]
        p_start, p_end = lo[split], hi[split]
        l_deep = level
    leaf_arr = np.sort(np.concatenate(leaves)) if leaves else np.zeros(0, np.int64)
    zmap = expand_zmap(leaf_arr, l_deep, l_max)
    return OracleIndex(mbr, th_quad, l_max, l_deep, leaf_arr, zmap,
                       trace if record_trace else None)


def expand_zmap(leaves: np.ndarray, l_deep: int, l_max: int) -> np.ndarray:
    """Run-length expansion of leaves in Morton order.  quadtree.py:142-158."""
    lv = leaves >> (2 * l_max)
    zz = leaves & ((1 << (2 * l_max)) - 1)
    span = np.left_shift(np.int64(1), 2 * (l_deep - lv))
    first = zz * span
    order = np.argsort(first, kind="stable")
    first, span = first[order], span[order]
    want = np.concatenate([[0], np.cumsum(span)[:-1]]) if len(span) else span
    if len(leaves) == 0 or np.any(first != want) or int(span.sum()) != 4 ** l_deep:
        raise OracleError("TilingGap", "leaves do not tile the grid")
    return np.repeat(leaves[order], span)


def map_objects(xs, ys, index: OracleIndex) -> np.ndarray:
    """Packed leaf per object via one zmap read.  quadtree.py:161-165."""
    i, j = cell_coords(xs, ys, index.mbr, index.l_deep)
    return index.zmap[morton(i, j)]


def leaf_occupancy(xs, ys, index: OracleIndex) -> np.ndarray:
    """Object count per leaf, aligned with index.leaves (quadtree.py:243-247)."""
    cells = map_objects(xs, ys, index)
    rows = np.searchsorted(index.leaves, cells)
    return np.bincount(rows, minlength=len(index.leaves)).astype(np.int64)


def needs_rebuild(xs, ys, index: OracleIndex, overfull_factor: float = 2.0, overfull_fraction: float = 0.05,
                  hard_factor: float = 8.0) -> bool:
    """quadtree.py:250-270: objects escaped the old MBR, any leaf over
    hard_factor * th_quad, or more than overfull_fraction of the leaves over
    overfull_factor * th_quad."""
    try:
        counts = leaf_occupancy(xs, ys, index)
    except OracleError as e:
        if e.kind == "OutOfBounds":
            return True
        raise
    if np.any(counts > hard_factor * index.th_quad):
        return True
    frac = float(np.mean(counts > overfull_factor * index.th_quad))
    return frac > overfull_fraction


def clip_rects(qxa, qya, qxb, qyb, mbr):
    """Intersect query rects with the index MBR; keep-mask of non-disjoint ones.

    grid.py:115-122 with geometry.py:80-88 (exact max/min, disjoint dropped).
    """
    xa = np.maximum(qxa, mbr[0])
    ya = np.maximum(qya, mbr[1])
    xb = np.minimum(qxb, mbr[2])
    yb = np.minimum(qyb, mbr[3])
    keep = ~((xa > xb) | (ya > yb))
    return keep, xa[keep], ya[keep], xb[keep], yb[keep]


@dataclass
class OracleSubqueries:
    qrow: np.ndarray  # row into the clipped query list
    cell: np.ndarray  # packed leaf id
    covering: np.ndarray  # bool


def split_queries(cxa, cya, cxb, cyb, index: OracleIndex) -> OracleSubqueries:
    """One subquery per (clipped query, intersected leaf).  quadtree.py:168-240.

    Level-synchronous implicit descent over the deepest-cell window (182-211),
    emission when the quadrant's first deepest cell belongs to a leaf no deeper
    than the quadrant (204-208); grouped stably per query (216-217); covering
    flag with the reference's exact op order (219-231).
    """
    m = len(cxa)
    if m == 0:
        e = np.zeros(0, np.int64)
        return OracleSubqueries(e, e.copy(), np.zeros(0, bool))
    mbr = index.mbr
    ld = index.l_deep
    i0, j0 = cell_coords(cxa, cya, mbr, ld)
    i1, j1 = cell_coords(cxb, cyb, mbr, ld)
    lvl_shift = 2 * index.l_max
    rows_out, leaf_out = [], []
    fr = np.arange(m, dtype=np.int64)
    fz = np.zeros(m, dtype=np.int64)
    for level in range(ld + 1):
        if len(fr) == 0:
            break
        span = 1 << (ld - level)
        fi, fj = unmorton(fz)
        ci, cj = fi * span, fj * span
        ok = (ci <= i1[fr]) & (ci + span - 1 >= i0[fr]) & (cj <= j1[fr]) & (cj + span - 1 >= j0[fr])
        fr, fz = fr[ok], fz[ok]
        probe = index.zmap[fz << (2 * (ld - level))]
        done = (probe >> lvl_shift) <= level
        rows_out.append(fr[done])
        leaf_out.append(probe[done])
        fr, fz = fr[~done], fz[~done]
        fr = np.repeat(fr, 4)
        fz = (np.repeat(fz, 4) << 2) | np.tile(np.arange(4, dtype=np.int64), len(fz))
    rows = np.concatenate(rows_out)
    cells = np.concatenate(leaf_out)
    order = np.argsort(rows, kind="stable")
    rows, cells = rows[order], cells[order]
    lev = cells >> lvl_shift
    li, lj = unmorton(cells & ((1 << lvl_shift) - 1))
    side = (np.int64(1) << lev).astype(np.float64)
    width = mbr[2] - mbr[0]
    height = mbr[3] - mbr[1]
    w = width / side
    h = height / side
    lxa = mbr[0] + li * w
    lya = mbr[1] + lj * h
    cov = ((cxa[rows] <= lxa) & (cxb[rows] >= np.minimum(lxa + w, mbr[2]))
           & (cya[rows] <= lya) & (cyb[rows] >= np.minimum(lya + h, mbr[3])))
    return OracleSubqueries(rows, cells, cov)


# --------------------------------------------------------------------------
# L3: per-cell directory
# --------------------------------------------------------------------------

@dataclass
class OracleDirectory:
    obj_order: np.ndarray  # input rows of objects in directory order
    obj_cell: np.ndarray
    isq_idx: np.ndarray  # indices into the subquery list, directory order
    cov_idx: np.ndarray
    cells: np.ndarray
    o_start: np.ndarray
    o_end: np.ndarray
    i_start: np.ndarray
    i_end: np.ndarray
    c_start: np.ndarray
    c_end: np.ndarray


def group_by_cell(obj_cell: np.ndarray, sq: OracleSubqueries) -> OracleDirectory:
    """Stable grouping of objects and subqueries per cell.  directory.py:119-158."""
    obj_order = np.argsort(obj_cell, kind="stable")
    oc = obj_cell[obj_order]
    sq_order = np.lexsort((sq.covering, sq.cell))
    isq_idx = sq_order[~sq.covering[sq_order]]
    cov_idx = sq_order[sq.covering[sq_order]]
    ic = sq.cell[isq_idx]
    cc = sq.cell[cov_idx]
    cells = np.unique(np.concatenate([oc, ic, cc]))
    return OracleDirectory(
        obj_order, oc, isq_idx, cov_idx, cells,
        np.searchsorted(oc, cells, "left"), np.searchsorted(oc, cells, "right"),
        np.searchsorted(ic, cells, "left"), np.searchsorted(ic, cells, "right"),
        np.searchsorted(cc, cells, "left"), np.searchsorted(cc, cells, "right"),
    )


# --------------------------------------------------------------------------
# L4: bitmaps (Alg. 2 + linearisation + popcounts)
# --------------------------------------------------------------------------

def cell_bitmap(oxs, oys, sxa, sya, sxb, syb) -> np.ndarray:
    """Linear (subquery-major) 32-bit words of one cell.

    bitmap.py:70-111: bit k of word b of subquery s <=> object 32b+k of the
    block satisfies xa<=x<=xb and ya<=y<=yb (89-94); padding bits zero (95-97);
    linear[s*blocks+b] (107).
    """
    nq, no = len(sxa), len(oxs)
    nb = -(no // -WORD_BITS)
    inside = ((oxs[None, :] >= sxa[:, None]) & (oxs[None, :] <= sxb[:, None])
              & (oys[None, :] >= sya[:, None]) & (oys[None, :] <= syb[:, None]))
    pad = np.zeros((nq, nb * WORD_BITS), dtype=bool)
    pad[:, :no] = inside
    return np.packbits(pad, axis=1, bitorder="little").view("<u4").reshape(-1).copy()


def word_popcounts(words: np.ndarray, nq: int) -> np.ndarray:
    """Per-subquery result counts.  bitmap.py:114-119."""
    if nq == 0:
        return np.zeros(0, np.int64)
    return np.bitwise_count(words.reshape(nq, -1)).sum(axis=1, dtype=np.int64)


def interlace(linear: np.ndarray, nq: int) -> np.ndarray:
    """Inverse of linearisation: interlaced[b*nq+s] == linear[s*nb+b].  bitmap.py:98,107."""
    nb = len(linear) // nq if nq else 0
    return np.ascontiguousarray(linear.reshape(nq, nb).T).reshape(-1)


# --------------------------------------------------------------------------
# Full tick
# --------------------------------------------------------------------------

@dataclass
class OracleTick:
    index: Optional[OracleIndex] = None
    keep: Optional[np.ndarray] = None  # per input query: survives clipping
    sub: Optional[OracleSubqueries] = None
    directory: Optional[OracleDirectory] = None
    obj_cell: Optional[np.ndarray] = None
    tasks: list = field(default_factory=list)  # (cell, o_rows, isq rows, linear words, counts)
    offsets: Optional[np.ndarray] = None  # CSR over input queries
    result_ids: Optional[np.ndarray] = None
    counters: dict = field(default_factory=dict)


def run_tick(ids, xs, ys, qids, qxa, qya, qxb, qyb, th_quad=384, l_max=L_MAX,
             covering_optimization=True, keep_tasks=False, index: Optional[OracleIndex] = None
             ) -> OracleTick:
    """One QUAD tick end to end (engine.py:178-259 with the quad branch).

    Returns the per-query results as a CSR in *input query order* (the
    reference keys them by issuer id in `ResultSet.by_query`; decode.py:102-123),
    each list ascending by object id.  `index` reuses a prebuilt index (the
    adaptive policy, engine.py:163-170).
    """
    ids = np.asarray(ids, np.int64)
    xs = np.asarray(xs, np.float64)
    ys = np.asarray(ys, np.float64)
    m = len(qids)
    out = OracleTick()
    if len(ids) == 0:  # engine.py:188-190
        out.offsets = np.zeros(m + 1, np.int64)
        out.result_ids = np.zeros(0, np.int64)
        return out
    if index is None:
        index = build_index(xs, ys, mbr_of(xs, ys), th_quad, l_max)
    out.index = index
    keep, cxa, cya, cxb, cyb = clip_rects(np.asarray(qxa, np.float64), np.asarray(qya, np.float64),
                                          np.asarray(qxb, np.float64), np.asarray(qyb, np.float64),
                                          index.mbr)
    out.keep = keep
    obj_cell = map_objects(xs, ys, index)
    sub = split_queries(cxa, cya, cxb, cyb, index)
    _join_decode(out, ids, xs, ys, m, keep, cxa, cya, cxb, cyb, obj_cell, sub, covering_optimization, keep_tasks)
    out.counters.update(n_leaves=int(len(index.leaves)), l_deep=int(index.l_deep))
    return out


def _join_decode(out, ids, xs, ys, m, keep, cxa, cya, cxb, cyb, obj_cell, sub, covering_optimization,
                 keep_tasks):
    """The index-independent part of a tick: directory, per-cell bitmaps,
    decode, covering expansion, canonical merge and counters
    (engine.py:199-259, 269-329).  Shared by the QUAD and UG methods."""
    out.obj_cell = obj_cell
    if not covering_optimization:  # engine.py:199-208
        sub = OracleSubqueries(sub.qrow, sub.cell, np.zeros(len(sub.cell), bool))
    out.sub = sub
    d = group_by_cell(obj_cell, sub)
    out.directory = d
    qrow_to_input = np.flatnonzero(keep)

    n_obj = d.o_end - d.o_start
    n_isq = d.i_end - d.i_start
    task_rows = np.flatnonzero((n_obj > 0) & (n_isq > 0))
    parts_q, parts_ids = [], []
    words_total = 0
    tests = 0
    for r in task_rows:
        orow = d.obj_order[d.o_start[r]:d.o_end[r]]
        srow = d.isq_idx[d.i_start[r]:d.i_end[r]]
        qr = sub.qrow[srow]
        words = cell_bitmap(xs[orow], ys[orow], cxa[qr], cya[qr], cxb[qr], cyb[qr])
        counts = word_popcounts(words, len(srow))
        nb = len(words) // len(srow)
        words_total += len(words)
        tests += len(srow) * len(orow)
        bits = np.unpackbits(words.reshape(len(srow), nb).view(np.uint8), axis=1,
                             bitorder="little")[:, :len(orow)]
        rr, cc = np.nonzero(bits)
        if np.any(np.bincount(rr, minlength=len(srow)) != counts):
            raise OracleError("CountMismatch", "decode disagrees with popcounts")
        parts_q.append(qrow_to_input[qr[rr]])
        parts_ids.append(ids[orow[cc]])
        if keep_tasks:
            out.tasks.append((int(d.cells[r]), orow, srow, words, counts))
    cov_results = 0
    for k in d.cov_idx:  # decode.py:83-99
        cell = sub.cell[k]
        r = np.searchsorted(d.cells, cell)
        orow = d.obj_order[d.o_start[r]:d.o_end[r]]
        if len(orow):
            parts_q.append(np.full(len(orow), qrow_to_input[sub.qrow[k]], np.int64))
            parts_ids.append(ids[orow])
            cov_results += len(orow)
    if parts_q:
        allq = np.concatenate(parts_q)
        alli = np.concatenate(parts_ids)
    else:
        allq = np.zeros(0, np.int64)
        alli = np.zeros(0, np.int64)
    # canonical per-query lists: group by input query, ascending id (decode.py:117)
    order = np.lexsort((alli, allq))
    allq, alli = allq[order], alli[order]
    dup = (allq[1:] == allq[:-1]) & (alli[1:] == alli[:-1])
    if np.any(dup):
        raise OracleError("DuplicateResult", "pair produced twice")
    counts_q = np.bincount(allq, minlength=m) if m else np.zeros(0, np.int64)
    out.offsets = np.concatenate([[0], np.cumsum(counts_q)]).astype(np.int64)
    out.result_ids = alli
    occ = n_obj[n_obj > 0]
    out.counters = dict(
        containment_tests=int(tests),
        decoded_bits=int(words_total) * WORD_BITS,
        subq_intersecting=int(len(d.isq_idx)),
        subq_covering=int(len(d.cov_idx)),
        covering_results=int(cov_results),
        active_cells=int(len(occ)),
        results_total=int(len(alli)),
        occupancy_mean=float(occ.mean()) if len(occ) else 0.0,
        occupancy_var=float(occ.var()) if len(occ) else 0.0,
    )


# --------------------------------------------------------------------------
# UG: the uniform-grid method (grid.py) over the same join / decode
# --------------------------------------------------------------------------

MAX_SPLIT_FACTOR = 1 << 16  # grid.py:22


def grid_axis_cells(values, origin: float, extent: float, n: int) -> np.ndarray:
    """floor((v - origin) * (n / extent)) clamped to n - 1; 0 when extent == 0.
    grid.py:42-46 (the scale is one Python float division, as there)."""
    values = np.asarray(values, np.float64)
    if extent > 0:
        return np.minimum((values - origin) * (n / extent), n - 1).astype(np.int64)
    return np.zeros(values.shape, np.int64)


def ug_map_objects(xs, ys, mbr, split_factor: int) -> np.ndarray:
    """Cell id = Morton(i, j) of the object's grid cell.  grid.py:55-68."""
    xa, ya, xb, yb = mbr
    xs = np.asarray(xs, np.float64)
    ys = np.asarray(ys, np.float64)
    if len(xs) and (np.any(xs < xa) or np.any(xs > xb) or np.any(ys < ya) or np.any(ys > yb)):
        raise OracleError("OutOfBounds", "object outside the grid MBR")
    i = grid_axis_cells(xs, xa, xb - xa, split_factor)
    j = grid_axis_cells(ys, ya, yb - ya, split_factor)
    return morton(i, j)


def ug_split_queries(cxa, cya, cxb, cyb, mbr, split_factor: int) -> OracleSubqueries:
    """One subquery per (clipped query, grid cell of its window), cells of a
    query in row-major order (i fastest), covering flag against the cell's
    extent inside the MBR.  grid.py:71-112."""
    xa, ya, xb, yb = mbr
    width, height = xb - xa, yb - ya
    cell_w = width / split_factor  # grid.py:39
    cell_h = height / split_factor
    i0 = grid_axis_cells(cxa, xa, width, split_factor)
    j0 = grid_axis_cells(cya, ya, height, split_factor)
    i1 = grid_axis_cells(cxb, xa, width, split_factor)
    j1 = grid_axis_cells(cyb, ya, height, split_factor)
    per = (i1 - i0 + 1) * (j1 - j0 + 1)
    if per.sum() == 0:
        return OracleSubqueries(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, bool))
    offs = np.concatenate([[0], np.cumsum(per)[:-1]])
    qrow = np.repeat(np.arange(len(per)), per)
    pos = np.arange(int(per.sum())) - offs[qrow]
    wdt = (i1 - i0 + 1)[qrow]
    ii = i0[qrow] + pos % wdt
    jj = j0[qrow] + pos // wdt
    lxa = xa + ii * cell_w
    lya = ya + jj * cell_h
    cov = ((cxa[qrow] <= lxa) & (cxb[qrow] >= np.minimum(lxa + cell_w, xb))
           & (cya[qrow] <= lya) & (cyb[qrow] >= np.minimum(lya + cell_h, yb)))
    return OracleSubqueries(qrow.astype(np.int64), morton(ii, jj), cov)


def ug_indexing_cost(d: OracleDirectory) -> int:
    """Containment tests + decoded bitmap bits over the task cells.  grid.py:125-138."""
    n_obj = d.o_end - d.o_start
    n_isq = d.i_end - d.i_start
    mask = (n_obj > 0) & (n_isq > 0)
    blocks = -(n_obj[mask] // -WORD_BITS)
    return int((n_isq[mask] * n_obj[mask]).sum()) + int((n_isq[mask] * blocks * WORD_BITS).sum())


def ug_sweep_costs(xs, ys, qxa, qya, qxb, qyb, candidates) -> list:
    """(split factor, cost) per candidate on one tick; the engine keeps the
    cheapest, ties to the smaller.  grid.py:141-165, engine.py:154-156."""
    xs = np.asarray(xs, np.float64)
    ys = np.asarray(ys, np.float64)
    mbr = mbr_of(xs, ys)
    keep, cxa, cya, cxb, cyb = clip_rects(np.asarray(qxa, np.float64), np.asarray(qya, np.float64),
                                          np.asarray(qxb, np.float64), np.asarray(qyb, np.float64), mbr)
    out = []
    for sf in candidates:
        oc = ug_map_objects(xs, ys, mbr, sf)
        sub = ug_split_queries(cxa, cya, cxb, cyb, mbr, sf)
        out.append((int(sf), ug_indexing_cost(group_by_cell(oc, sub))))
    return out


STAGING_CAPACITY = 1024  # baseline.py:17


def staging_flushes(tick: "OracleTick", capacity: int = STAGING_CAPACITY) -> int:
    """Shared-buffer flushes (= sync_ops) of the ug_baseline filter: per task cell
    a private stage of `capacity` pairs is flushed whenever full and once more
    for a partial remainder (baseline.py:64-103,106-121), i.e. ceil(pairs/capacity).
    Needs a tick run with keep_tasks=True."""
    total = 0
    for _, _, _, _, counts in tick.tasks:
        p = int(np.sum(counts))
        total += -(-p // capacity)
    return total


def run_tick_ug(ids, xs, ys, qids, qxa, qya, qxb, qyb, split_factor: int, covering_optimization=True,
                keep_tasks=False) -> OracleTick:
    """One UG tick end to end (engine.py:178-259 with the ug branch, 152-161)."""
    if not 1 <= split_factor <= MAX_SPLIT_FACTOR:
        raise OracleError("BadSplitFactor", str(split_factor))
    ids = np.asarray(ids, np.int64)
    xs = np.asarray(xs, np.float64)
    ys = np.asarray(ys, np.float64)
    m = len(qids)
    out = OracleTick()
    if len(ids) == 0:  # engine.py:188-190
        out.offsets = np.zeros(m + 1, np.int64)
        out.result_ids = np.zeros(0, np.int64)
        return out
    mbr = mbr_of(xs, ys)
    keep, cxa, cya, cxb, cyb = clip_rects(np.asarray(qxa, np.float64), np.asarray(qya, np.float64),
                                          np.asarray(qxb, np.float64), np.asarray(qyb, np.float64), mbr)
    out.keep = keep
    obj_cell = ug_map_objects(xs, ys, mbr, split_factor)
    sub = ug_split_queries(cxa, cya, cxb, cyb, mbr, split_factor)
    _join_decode(out, ids, xs, ys, m, keep, cxa, cya, cxb, cyb, obj_cell, sub, covering_optimization, keep_tasks)
    out.counters.update(split_factor=int(split_factor))
    return out


def brute_force(ids, xs, ys, qxa, qya, qxb, qyb):
    """Closed-rectangle scan per query over all objects.  oracle.py:17-28."""
    ids = np.asarray(ids, np.int64)
    offs = [0]
    parts = []
    for a, b, c, d in zip(qxa, qya, qxb, qyb):
        hit = (xs >= a) & (xs <= c) & (ys >= b) & (ys <= d)
        sel = np.sort(ids[hit])
        parts.append(sel)
        offs.append(offs[-1] + len(sel))
    res = np.concatenate(parts) if parts else np.zeros(0, np.int64)
    return np.asarray(offs, np.int64), res


def canonical_lines(qids, offsets, result_ids) -> list[str]:
    """`ResultSet.lines()` text for a CSR keyed by issuer (decode.py:33-37).

    Assumes unique issuer ids (one query per issuer per tick).
    """
    qids = np.asarray(qids, np.int64)
    order = np.argsort(qids, kind="stable")
    lines = []
    for q in order:
        seg = result_ids[offsets[q]:offsets[q + 1]]
        lines.append(f"{int(qids[q])}: {','.join(str(int(v)) for v in seg)}".rstrip())
    return lines


def digest_lines(lines: list[str]) -> str:
    h = hashlib.sha256()
    for ln in lines:
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


def result_digest(qids, offsets, result_ids) -> str:
    """sha256 of the canonical lines — the compact pin used for large goldens."""
    return digest_lines(canonical_lines(qids, offsets, result_ids))
