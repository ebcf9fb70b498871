"""Multi-GPU orchestration on CPU: world_size 2 (and 3) over gloo.

distributed_estimate shards SEGMENTS across ranks, reduce-scatters the partial
raw sums by line blocks (padded), exchanges the w-1 line halo, smooths each
rank's output rows and all-gathers the lexicographic slices.
Here the compute hooks are a CPU engine written independently from the D_h
definition, so this checks the collective plumbing and the layout bookkeeping;
the GPU hooks (hos_partial_raw / hos_smooth_raw) are checked against the same
bookkeeping on one GPU in test_gpu_parity.py::test_shard_pipeline_single_gpu.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hos_oracle as O


class CpuEngine:
    """Raw-sum and smoothing hooks on the host (order 3), CSR line layout."""

    def __init__(self, m, k, w, conj, x, taper):
        h = w // 2
        self.m, self.k, self.w, self.conj = m, k, w, conj
        self.lo, self.hi = -h, w - 1 - h
        rows = (m - 1) // 2 + 1
        stop = [min(k1, (m - 2 * k1 - 1) // 2) + 1 for k1 in range(rows)]
        self.cmax = [max(stop[kk] - 1 for kk in range(max(0, a - self.hi), min(rows - 1, a - self.lo) + 1)) + self.hi
                     for a in range(self.lo, rows + self.hi)]
        self.line_start = np.concatenate([[0], np.cumsum([c - self.lo + 1 for c in self.cmax])]).astype(np.int64)
        self.row_off = np.concatenate([[0], np.cumsum(stop)]).astype(np.int64)
        self.stop = stop
        self.spec = O.segment_spectra(x, m, k, taper)

    def rows_line_range(self, r0, r1):
        return (r0, r1 + self.w - 1) if r1 > r0 else (r0, r0)

    def partial_raw(self, x, s0, s1):
        F = self.spec[s0:s1]
        G = np.conj(F) if self.conj else F
        raw = np.zeros(int(self.line_start[-1]), np.complex128)
        for line, cm in enumerate(self.cmax):
            a = self.lo + line
            b = np.arange(self.lo, cm + 1)
            vals = (F[:, a % self.m][:, None] * F[:, b % self.m] * G[:, (a + b) % self.m]).sum(axis=0)
            raw[self.line_start[line]: self.line_start[line + 1]] = vals
        return torch.from_numpy(raw)

    def smooth(self, local, line_begin, r0, r1):
        local = local.numpy()
        base = self.line_start[line_begin]
        out = []
        for k1 in range(r0, r1):
            for k2 in range(self.stop[k1]):
                s = 0j
                for u in range(self.lo, self.hi + 1):
                    line = k1 + u - self.lo
                    c0 = self.line_start[line] - base
                    s += local[c0 + k2: c0 + k2 + self.w].sum()
                out.append(s / (self.m * self.k * self.w ** 2))
        return torch.tensor(np.asarray(out, np.complex128))

    def zeros(self, n, dtype):
        return torch.zeros(n, dtype=dtype)

    def as_real(self, t):
        return torch.view_as_real(t).reshape(-1)

    def from_real(self, t):
        return torch.view_as_complex(t.reshape(-1, 2))

    def backend_supports_rs(self, group):
        return False


def _worker(rank, world, port, cfgs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_11775_b200 import EstimationConfig, SegmentConfig, distributed_estimate

        res = []
        for m, k, w, conj, seed in cfgs:
            x = np.random.default_rng(seed).standard_normal(m * k)
            cfg = EstimationConfig(3, SegmentConfig(m=m, k=k), w, conjugate_last=conj, taper="hann")
            eng = CpuEngine(m, k, w, conj, x, "hann")
            vals = distributed_estimate(x, cfg, engine=eng).numpy()
            part, (p0, p1) = distributed_estimate(x, cfg, engine=eng, gather=False)
            res.append((vals, part.numpy(), p0, p1))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CFGS = [(64, 6, 5, True, 1), (48, 5, 4, False, 2), (128, 3, 9, True, 3)]


@pytest.mark.parametrize("world", [2, 3])
def test_segment_sharded_estimate_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CFGS, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, (m, k, w, conj, seed) in enumerate(CFGS):
        x = np.random.default_rng(seed).standard_normal(m * k)
        _, ref = O.estimate(x, 3, m, k, w, conj, "hann")
        scale = np.abs(ref).max()
        slices = []
        for r in range(world):
            vals, part, p0, p1 = out[r][i]
            assert np.max(np.abs(vals - ref)) <= 1e-12 * scale, (world, r, i)
            slices.append((p0, p1, part))
        slices.sort()
        assert slices[0][0] == 0 and slices[-1][1] == len(ref)
        for (a0, a1, part), (b0, _, _) in zip(slices, slices[1:] + [(len(ref), 0, None)]):
            assert a1 == b0 and len(part) == a1 - a0
            assert np.max(np.abs(part - ref[a0:a1]), initial=0.0) <= 1e-12 * scale


def _oracle_rows(rows, cfg):
    """CPU engine for sharded_batch_estimate: the oracle on each series."""
    vals = [O.estimate(r, cfg.order, cfg.segment.m, cfg.segment.k, cfg.m3, cfg.conjugate_last, cfg.taper)[1]
            for r in rows]
    return torch.from_numpy(np.stack(vals))


def _series_worker(rank, world, port, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_11775_b200 import EstimationConfig, SegmentConfig, sharded_batch_estimate

        x = np.random.default_rng(77).standard_normal((batch, 64 * 3))
        cfg = EstimationConfig(3, SegmentConfig(m=64, k=3), 5, taper="hann")
        calls = []
        eng = lambda rows, c: (calls.append(len(rows)), _oracle_rows(rows, c))[1]
        full = sharded_batch_estimate(x, cfg, engine=eng).numpy()
        part, (b0, b1) = sharded_batch_estimate(x, cfg, engine=eng, gather=False)
        q.put((rank, full, None if part is None else part.numpy(), b0, b1, calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,batch", [(2, 7), (3, 8), (2, 1)])
def test_series_sharded_batch_gloo(world, batch):
    """Batched series split by series (north_star: no collective on the data
    path): every rank computes only its contiguous series range, the ranges
    tile the batch, and the gathered (batch, npoints) result equals the
    oracle row by row."""
    from paper_1805_11775_b200 import series_shard

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_series_worker, args=(r, world, port, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {r: rest for r, *rest in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = np.random.default_rng(77).standard_normal((batch, 64 * 3))
    ref = np.stack([O.estimate(r, 3, 64, 3, 5, True, "hann")[1] for r in x])
    covered = []
    for r in range(world):
        full, part, b0, b1, calls = out[r]
        assert (b0, b1) == series_shard(batch, r, world)
        assert np.array_equal(full, ref)
        assert calls == ([b1 - b0] * 2 if b1 > b0 else [])  # only its own series, never the batch
        if b1 > b0:
            assert np.array_equal(part, ref[b0:b1])
        covered += list(range(b0, b1))
    assert covered == list(range(batch))
