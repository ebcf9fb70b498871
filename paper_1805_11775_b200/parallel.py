"""Data-parallel estimation (drop-in for hospectra/parallel.py) and the
multi-GPU segment-sharded path.

``parallel_estimate`` keeps the reference contract (same values for every
worker count, parallel.py:120-162): on one GPU the worker count does not
change the computation at all, so the result is bit-identical for any
``WorkerConfig``.  ``partition_domain`` keeps the reference's row_blocks /
point_blocks semantics (parallel.py:62-91) and is reused to cut output rows
across GPUs.

``distributed_estimate`` is the B200 multi-GPU path: one
process per GPU, segments sharded across ranks, each rank computes partial
raw sums over the whole dilated domain D_h (hos_partial_raw), the partials
are reduce-scattered by contiguous line blocks (padded to a common count,
as NCCL requires), each rank fetches the w-1 lines of halo it needs from the
next rank (one send/recv pair per neighbour), smooths its own output rows
(hos_smooth_raw) and the lexicographic slices are all-gathered.  The
collective plumbing is torch.distributed (NCCL on GPUs, gloo in the CPU
tests); the compute hooks are injectable so the orchestration is tested on
CPU with world_size 2.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError
from .series import TimeSeries
from .spectra import EstimationConfig, SpectrumGrid, estimate_spectrum, principal_domain

__all__ = ["WorkerConfig", "partition_domain", "parallel_estimate", "row_blocks", "ShardLayout",
           "shard_layout", "distributed_estimate", "series_shard", "sharded_batch_estimate"]


@dataclass(frozen=True)
class WorkerConfig:
    """Worker count and output-partition strategy (hospectra/parallel.py:40-59)."""

    p: int = 1
    partition: str = "row_blocks"

    def __post_init__(self):
        if self.p < 1:
            raise ParameterError(f"worker count must be >= 1, got {self.p}")
        if self.partition not in ("row_blocks", "point_blocks"):
            raise ParameterError(
                f"partition must be 'row_blocks' or 'point_blocks', got {self.partition!r}")


def _split_bounds(dom: np.ndarray, workers: WorkerConfig) -> list[int]:
    total = len(dom)
    p = workers.p
    if p == 1 or total == 0:
        return [0, total] + [total] * (p - 1)
    if workers.partition == "point_blocks":
        q, r = divmod(total, p)
        sizes = [q + 1] * r + [q] * (p - r)
        return [0] + [int(v) for v in np.cumsum(sizes)]
    _, first, counts = np.unique(dom[:, 0], return_index=True, return_counts=True)
    cum = np.cumsum(counts)
    targets = np.arange(1, p) * (total / p)
    gb = np.searchsorted(cum, targets, side="left") + 1
    cuts = [int(first[b]) if b < len(first) else total for b in gb]
    return [0] + cuts + [total]


def partition_domain(domain, workers: WorkerConfig) -> list:
    """Disjoint contiguous parts of a lex-ordered domain whose concatenation
    is the input (hospectra/parallel.py:83-91)."""
    dom = np.asarray(domain)
    b = _split_bounds(dom, workers)
    return [dom[b[i]: b[i + 1]] for i in range(workers.p)]


def parallel_estimate(series: TimeSeries, cfg: EstimationConfig, workers: WorkerConfig, *,
                      device=None, devices=None) -> SpectrumGrid:
    """Same contract as ``estimate_spectrum`` for every worker count
    (hospectra/parallel.py:120-162), with ``workers.p`` mapped to GPUs.

    ``p == 1`` (or one visible GPU): the whole estimate on one device, values
    identical for every ``WorkerConfig``.  ``p > 1`` with several GPUs: the
    K-sum is split across ``g = min(p, device_count)`` devices of this process
    by contiguous segment ranges: every device runs the front
    end + triple product on its segments (``hos_partial_raw``), the partial
    raw sums are added on the first device in device order (fixed, so the
    result is deterministic for a given g), and that device smooths the whole
    grid (``hos_smooth_raw``).  Across different g the values agree within the
    precision's parity bar (the segment sum is regrouped).  ``devices``
    overrides the device list (tests: several shards on one GPU)."""
    if not isinstance(workers, WorkerConfig):
        raise ParameterError("workers must be a WorkerConfig")
    cfg.segment.validate_for(series)
    import torch

    if devices is None:
        n_dev = torch.cuda.device_count() if torch.cuda.is_available() else 0
        g = min(workers.p, n_dev)
        base = 0 if device is None else int(device)
        devices = [(base + i) % max(n_dev, 1) for i in range(g)]
    devices = list(devices)
    if len(devices) <= 1:
        return estimate_spectrum(series, cfg, device=devices[0] if devices else device)
    return _segment_split_estimate(series, cfg, devices)


def _segment_split_estimate(series: TimeSeries, cfg: EstimationConfig, devices) -> SpectrumGrid:
    import torch

    from ._native import get_plan

    k, m = cfg.segment.k, cfg.segment.m
    g = len(devices)
    segb = [(r * k) // g for r in range(g + 1)]
    xs = np.ascontiguousarray(series.samples[: k * m])
    raws = []
    for r, d in enumerate(devices):  # launches are asynchronous: the devices run concurrently
        plan = get_plan(cfg.order, m, k, cfg.m3, cfg.conjugate_last, cfg.bits, cfg.taper, 1, d)
        with torch.cuda.device(d):
            x = torch.from_numpy(xs).to(f"cuda:{d}")
            raw = torch.empty(plan.cells, dtype=plan.complex_dtype, device=f"cuda:{d}")
            raws.append(plan.partial_raw(x, segb[r], segb[r + 1], raw))
    d0 = devices[0]
    plan0 = get_plan(cfg.order, m, k, cfg.m3, cfg.conjugate_last, cfg.bits, cfg.taper, 1, d0)
    with torch.cuda.device(d0):
        total = raws[0].clone()
        for raw in raws[1:]:  # fixed device order
            total += raw.to(f"cuda:{d0}")
        rows = (m - 1) // 2 + 1
        out = torch.empty(plan0.npoints, dtype=plan0.complex_dtype, device=f"cuda:{d0}")
        plan0.smooth_raw(total, 0, 0, rows, out)
        vals = out.cpu().numpy().astype(np.complex128, copy=False)
    return SpectrumGrid(order=cfg.order, m=m, m3=cfg.m3, plan=cfg.plan,
                        indices=principal_domain(cfg.order, m), values=vals)


# ---------------------------------------------------------------------------
# multi-GPU: batches of independent series, sharded by series (no collective)


def series_shard(batch: int, rank: int, nranks: int) -> tuple:
    """Contiguous, balanced series range [b0, b1) of ``rank``."""
    if not (0 <= rank < nranks):
        raise ParameterError(f"rank {rank} outside [0, {nranks})")
    return (rank * batch) // nranks, ((rank + 1) * batch) // nranks


def sharded_batch_estimate(x, cfg: EstimationConfig, *, group=None, gather: bool = True, engine=None):
    """Independent estimates of the rows of ``x`` (batch, n), split by series
    across the ranks of ``group`` (one process per GPU).  Each rank computes
    only its own rows [b0, b1) -- there is no collective on the data path
    (north_star: "multi-series batches shard by series with no collective").
    ``gather=True`` collects the (batch, npoints) values on every rank (one
    all-gather of padded shards, the analogue of hospectra/parallel.py:155's
    shared result buffer); ``gather=False`` returns (values of [b0, b1), (b0, b1)).
    ``engine(x_rows, cfg)`` computes a shard (default: estimate_batch on the
    current GPU); the CPU tests inject one."""
    import torch
    import torch.distributed as dist

    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    batch = x.shape[0]
    b0, b1 = series_shard(batch, rank, nranks)
    if engine is None:
        from .spectra import estimate_batch

        engine = lambda rows, c: estimate_batch(rows, c, to_host=False)
    vals = engine(x[b0:b1], cfg) if b1 > b0 else None
    if not gather:
        return vals, (b0, b1)
    npts = len(principal_domain(cfg.order, cfg.segment.m))
    width = max(series_shard(batch, r, nranks)[1] - series_shard(batch, r, nranks)[0] for r in range(nranks))
    like = vals if vals is not None else torch.zeros(0)
    dev = like.device if isinstance(like, torch.Tensor) else torch.device("cpu")
    dt = like.dtype if isinstance(like, torch.Tensor) and like.numel() else torch.complex128
    pad = torch.zeros((max(width, 1), npts), dtype=dt, device=dev)
    if vals is not None:
        pad[: b1 - b0] = torch.as_tensor(vals, device=dev).reshape(b1 - b0, npts)
    real = torch.view_as_real(pad).reshape(-1)
    outs = [torch.empty_like(real) for _ in range(nranks)]
    dist.all_gather(outs, real, group=group)
    res = torch.empty((batch, npts), dtype=dt, device=dev)
    for r in range(nranks):
        a, b = series_shard(batch, r, nranks)
        if b > a:
            res[a:b] = torch.view_as_complex(outs[r].reshape(-1, npts, 2))[: b - a]
    return res


# ---------------------------------------------------------------------------
# multi-GPU: segment sharding + reduce-scatter + halo


def row_blocks(row_off: np.ndarray, nranks: int) -> list[int]:
    """Output-row cut points [r_0=0, ..., r_P=rows] balancing point counts at
    whole-row granularity (the row_blocks policy of parallel.py:73-80)."""
    rows = len(row_off) - 1
    total = int(row_off[-1])
    if nranks == 1 or total == 0:
        return [0] + [rows] * nranks
    counts = np.diff(row_off)
    cum = np.cumsum(counts)
    targets = np.arange(1, nranks) * (total / nranks)
    cuts = [int(min(rows, np.searchsorted(cum, t, side="left") + 1)) for t in targets]
    return [0] + cuts + [rows]


@dataclass
class ShardLayout:
    """Who owns which lines/cells and output points."""

    nranks: int
    seg_bounds: list          # segment shard [s_r, s_{r+1})
    row_bounds: list          # output rows [r_r, r_{r+1})
    own_lines: list           # (l0, l1) lines reduce-scattered to rank r
    need_lines: list          # (l0, l1) lines rank r smooths from
    own_cells: list           # (c0, c1)
    need_cells: list          # (c0, c1)
    point_bounds: list        # lexicographic [p_r, p_{r+1})
    block: int                # padded reduce-scatter block (cells)
    halo: int                 # padded halo length (cells)
    halo_in_next: bool        # every rank's halo lies in rank r+1's block


def shard_layout(k: int, row_off: np.ndarray, line_start: np.ndarray, rows_line_range, nranks: int) -> ShardLayout:
    """Static partition: segments evenly, output rows by row_blocks, lines
    owned from the first line of each rank's rows, halo = lines the rank's
    rows need past its own block."""
    segb = [(r * k) // nranks for r in range(nranks + 1)]
    rb = row_blocks(row_off, nranks)
    nlines = len(line_start) - 1
    need = [rows_line_range(rb[r], rb[r + 1]) for r in range(nranks)]
    starts = []
    for r in range(nranks):
        lb = need[r][0] if rb[r] < rb[r + 1] else None
        starts.append(lb)
    # owned blocks: from each rank's first needed line to the next rank's
    own = []
    nxt = nlines
    for r in reversed(range(nranks)):
        l0 = starts[r] if starts[r] is not None else nxt
        own.append((l0, nxt))
        nxt = l0
    own.reverse()
    own[0] = (0, own[0][1])  # rank 0 owns from the first line (lines before are unused)
    need_lines = [(need[r][0], need[r][1]) if rb[r] < rb[r + 1] else (own[r][0], own[r][0])
                  for r in range(nranks)]
    cells = lambda l0, l1: (int(line_start[l0]), int(line_start[l1]))
    own_cells = [cells(*o) for o in own]
    need_cells = [cells(*n) for n in need_lines]
    block = max(max(c1 - c0 for c0, c1 in own_cells), 1)
    halos = [max(0, need_cells[r][1] - own_cells[r][1]) for r in range(nranks)]
    halo = max(max(halos), 1)
    in_next = all(halos[r] == 0 or (r + 1 < nranks and halos[r] <= own_cells[r + 1][1] - own_cells[r + 1][0])
                  for r in range(nranks))
    pb = [int(row_off[r]) for r in rb]
    return ShardLayout(nranks, segb, rb, own, need_lines, own_cells, need_cells, pb, block, halo, in_next)


def distributed_estimate(x, cfg: EstimationConfig, *, group=None, engine=None, gather: bool = True):
    """Segment-sharded estimate of ONE series across the ranks of ``group``.

    ``x``: the full series on every rank (host numpy or a CUDA tensor; each
    rank only reads its own segments).  ``engine`` supplies the compute
    hooks (default: the GPU library); tests inject a CPU engine.
    Returns the full (npoints,) value vector on every rank when ``gather``,
    else this rank's lexicographic slice and its point range."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    nranks = dist.get_world_size(group)
    if engine is None:
        engine = _GpuEngine(cfg)
    lay = shard_layout(cfg.segment.k, engine.row_off, engine.line_start, engine.rows_line_range, nranks)
    s0, s1 = lay.seg_bounds[rank], lay.seg_bounds[rank + 1]
    raw = engine.partial_raw(x, s0, s1)                      # (ncells,) complex partial sums
    send = engine.zeros(nranks * lay.block, raw.dtype)
    for r in range(nranks):
        c0, c1 = lay.own_cells[r]
        send[r * lay.block: r * lay.block + (c1 - c0)] = raw[c0:c1]
    mine = engine.zeros(lay.block, raw.dtype)
    _reduce_scatter(dist, engine, mine, send, group)
    oc0, oc1 = lay.own_cells[rank]
    nc0, nc1 = lay.need_cells[rank]
    local = engine.zeros(max(nc1, oc1) - oc0, raw.dtype)
    local[: oc1 - oc0] = mine[: oc1 - oc0]
    # halo: lines past the owned block, held by the following rank(s)
    if lay.halo_in_next:
        # one send/recv pair per neighbour: rank r+1 sends the head of its
        # block (the w-1 lines rank r's rows read past its own block)
        need = max(0, nc1 - oc1)
        need_prev = max(0, lay.need_cells[rank - 1][1] - lay.own_cells[rank - 1][1]) if rank > 0 else 0
        # gloo moves point-to-point messages between host tensors only
        host = dist.get_backend(group) == "gloo"
        stage = (lambda t: t.cpu()) if host else (lambda t: t)
        ops = []
        recv_buf = stage(engine.zeros(max(need, 1), raw.dtype))
        if need:
            ops.append(dist.P2POp(dist.irecv, engine.as_real(recv_buf), _global_rank(dist, group, rank + 1), group))
        if need_prev:
            ops.append(dist.P2POp(dist.isend, engine.as_real(stage(mine[:need_prev]).clone()),
                                  _global_rank(dist, group, rank - 1), group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if need:
            local[oc1 - oc0: oc1 - oc0 + need] = recv_buf[:need].to(local.device)
    else:
        blocks = _all_gather(dist, engine, mine, nranks, group)
        for r in range(rank + 1, nranks):
            c0, c1 = lay.own_cells[r]
            lo_, hi_ = max(c0, oc1), min(c1, nc1)
            if lo_ < hi_:
                local[lo_ - oc0: hi_ - oc0] = blocks[r][lo_ - c0: hi_ - c0]
    r0, r1 = lay.row_bounds[rank], lay.row_bounds[rank + 1]
    vals = engine.smooth(local, lay.own_lines[rank][0], r0, r1)  # points [p_r, p_{r+1})
    if not gather:
        return vals, (lay.point_bounds[rank], lay.point_bounds[rank + 1])
    pmax = max(lay.point_bounds[r + 1] - lay.point_bounds[r] for r in range(nranks))
    pad = engine.zeros(max(pmax, 1), vals.dtype)
    pad[: len(vals)] = vals
    parts = _all_gather(dist, engine, pad, nranks, group)
    out = engine.zeros(lay.point_bounds[-1], vals.dtype)
    for r in range(nranks):
        a, b = lay.point_bounds[r], lay.point_bounds[r + 1]
        out[a:b] = parts[r][: b - a]
    return out


_NATIVE = {}


def native_distributed_plan(cfg: EstimationConfig, group=None):
    """The library's own multi-GPU path (hos_comm_attach + hos_estimate_
    distributed: NCCL reduce-scatter / all-gather issued inside the C-ABI, no
    per-step Python collectives): a plan of ``cfg`` on the current device with
    a dedicated NCCL communicator over the ranks of ``group``, built once per
    (cfg, device, group).  The communicator's unique id travels over
    ``torch.distributed`` (broadcast from rank 0).  Use ``plan.estimate_
    distributed(x)`` with the full series on every rank."""
    import ctypes

    import torch
    import torch.distributed as dist

    from ._native import get_plan

    dev = torch.cuda.current_device()
    key = (cfg.order, cfg.segment.m, cfg.segment.k, cfg.m3, cfg.conjugate_last, cfg.bits, cfg.taper, dev, id(group))
    if key in _NATIVE:
        return _NATIVE[key][0]
    nccl = ctypes.CDLL("libnccl.so.2")

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_byte * 128)]

    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    uid = UniqueId()
    buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        if nccl.ncclGetUniqueId(ctypes.byref(uid)) != 0:
            raise RuntimeError("ncclGetUniqueId failed")
        buf.copy_(torch.frombuffer(bytearray(bytes(uid.internal)), dtype=torch.uint8))
    dist.broadcast(buf, 0, group=group)
    ctypes.memmove(ctypes.byref(uid), bytes(buf.cpu().numpy().tobytes()), 128)
    comm = ctypes.c_void_p()
    rc = nccl.ncclCommInitRank(ctypes.byref(comm), nranks, uid, rank)
    if rc != 0:
        raise RuntimeError(f"ncclCommInitRank failed ({rc})")
    plan = get_plan(cfg.order, cfg.segment.m, cfg.segment.k, cfg.m3, cfg.conjugate_last, cfg.bits, cfg.taper, 1, dev)
    plan.comm_attach(comm.value, rank, nranks)
    _NATIVE[key] = (plan, nccl, comm)
    return plan


def _global_rank(dist, group, r):
    return r if group is None else dist.get_global_rank(group, r)


def _reduce_scatter(dist, engine, out, inp, group):
    # complex -> real view (NCCL/gloo reduce real dtypes)
    o, i = engine.as_real(out), engine.as_real(inp)
    if hasattr(dist, "reduce_scatter_tensor") and engine.backend_supports_rs(group):
        dist.reduce_scatter_tensor(o, i, group=group)
    else:
        # gloo has no reduce_scatter: all_reduce then slice (CPU tests only)
        tmp = i.clone()
        dist.all_reduce(tmp, group=group)
        r = dist.get_rank(group)
        n = o.numel()
        o.copy_(tmp[r * n: (r + 1) * n])


def _all_gather(dist, engine, t, nranks, group):
    import torch

    rt = engine.as_real(t)
    outs = [torch.empty_like(rt) for _ in range(nranks)]
    dist.all_gather(outs, rt, group=group)
    return [engine.from_real(o) for o in outs]


class _GpuEngine:
    """Compute hooks backed by libhos_b200 on the current CUDA device."""

    def __init__(self, cfg: EstimationConfig):
        import torch

        from ._native import get_plan

        self.torch = torch
        self.cfg = cfg
        self.plan = get_plan(cfg.order, cfg.segment.m, cfg.segment.k, cfg.m3, cfg.conjugate_last, cfg.bits,
                             cfg.taper, 1, torch.cuda.current_device())
        self.line_start = self.plan.line_starts()
        rows = (cfg.segment.m - 1) // 2 + 1
        self.row_off = np.array([self.plan.row_point_offset(r) for r in range(rows + 1)], dtype=np.int64)
        self.rows_line_range = self.plan.rows_line_range
        self.device = torch.device("cuda", self.plan.device)

    def partial_raw(self, x, s0, s1):
        torch = self.torch
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x)).to(self.device)
        raw = torch.empty(self.plan.cells, dtype=self.plan.complex_dtype, device=self.device)
        return self.plan.partial_raw(x, s0, s1, raw)

    def smooth(self, local, line_begin, r0, r1):
        torch = self.torch
        n = self.plan.row_point_offset(r1) - self.plan.row_point_offset(r0)
        out = torch.empty(max(n, 1), dtype=self.plan.complex_dtype, device=self.device)
        if n:
            self.plan.smooth_raw(local, line_begin, r0, r1, out)
        return out[:n]

    def zeros(self, n, dtype):
        return self.torch.zeros(n, dtype=dtype, device=self.device)

    def as_real(self, t):
        return self.torch.view_as_real(t).reshape(-1)

    def from_real(self, t):
        return self.torch.view_as_complex(t.reshape(-1, 2))

    def backend_supports_rs(self, group):
        import torch.distributed as dist

        return dist.get_backend(group) == "nccl"
