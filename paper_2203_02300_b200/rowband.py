"""Row-band frames: one frame split over G ranks (BASELINE config D,
3840x2160 D=256 "row-band partitioning with halo exchange over NVLink").

Per composited frame (pipeline.cpp:183-258), band k of G:
  * stereo on its quarter rows plus the recompute halo (dco_stereo_band); the
    aggregation column prefix arrives from band k-1 and leaves for band k+1
    (the chain is the one true data exchange of the stereo stage);
  * flow, amplitude fusion, box filter, normalisation, blur and contours run
    on the whole frame on every rank (they are 5 % of a 4K frame, and the
    global maxima of contour.cpp:139-141/197-200 and the hysteresis flood then
    need no exchange);
  * the frame-wide sparse mean is combined from every band's exact partial
    sums (dco_band_sparse_mean), then each band assembles its full rows plus a
    2-row halo (dco_band_assemble);
  * the PCG + MR solve runs over all bands at once (dco_band_solver: reduction
    and p halo through peer memory inside one persistent kernel per GPU);
  * each band composites its own rows.

Links: LocalLinks runs all G bands in this process on one GPU (the solve as
one cooperative launch over all bands); DistLinks gives each rank one band and
moves the carries, the sparse statistics and the solver handles with
torch.distributed (NCCL on GPUs). The band code is the same for both.
"""
import math

import torch

from . import dco
from .config import Config, UnsolvableFrameError


class LocalLinks:
    """Every band in this process (fewer GPUs than bands)."""

    def __init__(self, bands):
        self.bands = bands
        self.owned = list(range(bands))
        self._carry = {}

    def put_carry(self, key, t):
        k, d0 = key
        self._carry[(k + 1, d0)] = t

    def get_carry(self, key, like):
        return self._carry.pop(key)

    def gather_stats(self, stats):
        return [stats[k] for k in range(self.bands)]

    def gather_bytes(self, blobs):
        return [blobs[k] for k in range(self.bands)]

    def gather_rows(self, rows):
        """Every band's rows, stacked in band (= row) order."""
        return torch.cat([rows[k] for k in range(self.bands)], dim=0)


class DistLinks:
    """One band per rank over torch.distributed (rank k owns band k)."""

    def __init__(self, group_dist, world, rank, device=None):
        self.dist = group_dist
        self.bands = world
        self.rank = rank
        self.owned = [rank]
        self.device = device

    def put_carry(self, key, t):
        self.dist.send(t, dst=key[0] + 1)

    def get_carry(self, key, like):
        t = torch.empty_like(like)
        self.dist.recv(t, src=key[0] - 1)
        return t

    def gather_stats(self, stats):
        mine = torch.tensor(stats[self.rank], dtype=torch.float64, device=self.device)
        out = [torch.empty_like(mine) for _ in range(self.bands)]
        self.dist.all_gather(out, mine)
        return [o.tolist() for o in out]

    def gather_bytes(self, blobs):
        out = [None] * self.bands
        self.dist.all_gather_object(out, blobs[self.rank])
        return out

    def gather_rows(self, rows):
        """Every rank's band rows, stacked in band order (bands differ in
        height: padded to the tallest for the all_gather, then trimmed)."""
        mine = rows[self.rank]
        heights = self.gather_stats({self.rank: [float(mine.shape[0]), 0.0, 0.0, 0.0]})
        hmax = int(max(h[0] for h in heights))
        pad = torch.zeros((hmax,) + tuple(mine.shape[1:]), dtype=mine.dtype, device=mine.device)
        pad[: mine.shape[0]] = mine
        out = [torch.empty_like(pad) for _ in range(self.bands)]
        self.dist.all_gather(out, pad)
        return torch.cat([o[: int(h[0])] for o, h in zip(out, heights)], dim=0)


class RowBandFrames:
    """The row-band frame loop of one stream: owns the band plans, the band
    solvers and the previous dense rows (the d_pre chain, pipeline.cpp:133,235)."""

    def __init__(self, full_w, full_h, cfg: Config, links, chunk=None):
        """chunk: slices per carry message (a multiple of 32); default 32 with
        one band per rank, the whole range when all bands share this GPU."""
        self.fw, self.fh, self.cfg, self.links = full_w, full_h, cfg, links
        self.chunk = chunk if chunk is not None else (32 if isinstance(links, DistLinks) else None)
        g = links.bands
        self.plans = {k: dco.band_plan(cfg, full_w, full_h, g, k) for k in links.owned}
        self.solvers = {}
        for k, b in self.plans.items():
            self.solvers[k] = dco.BandSolver(g, k, full_w, b.frow0, b.frow1 - b.frow0, full_h)
        if isinstance(links, LocalLinks):
            dco.band_connect_local([self.solvers[k] for k in range(g)])
        else:
            handles = links.gather_bytes({k: s.export() for k, s in self.solvers.items()})
            for s in self.solvers.values():
                s.connect(handles)
        self.prev = {}  # band -> dense rows of the previous frame
        self.iterations = 0
        self.timing = False  # CUDA-event spans per phase into self.spans (ms, summed)
        self.spans = {}
        self._marks = []

    def _mark(self, name):
        if self.timing:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self._marks.append((name, e))

    def _close_marks(self):
        if not self.timing or not self._marks:
            return
        torch.cuda.synchronize()
        for (_, a), (name, b) in zip(self._marks, self._marks[1:]):
            self.spans[name] = self.spans.get(name, 0.0) + a.elapsed_time(b)
        self._marks = []

    def close(self):
        for s in self.solvers.values():
            s.close()
        self.solvers = {}

    force_sequential_mean = False  # tests: take the gathered sequential mean even inside the guard

    def _sub(self, b):
        """Full rows of a band's assembly sub-frame: owned + 2 (even start)."""
        return max(0, b.frow0 - 2), min(self.fh, b.frow1 + 2)

    def frame(self, past_q, mid_q, future_q, mid_gray, right_q, mid_rgb, vrgb=None, vdepth=None):
        """One composited frame. Inputs are whole-frame device tensors (quarter
        lefts of the keyframe window, the middle frame's gray, right quarter and
        RGB; optional virtual layer). Returns {band: dict(dense, composite,
        mask, sparse, rows)} for the bands this process owns."""
        cfg, fw, fh, L = self.cfg, self.fw, self.fh, self.links
        self._mark("start")
        # whole-frame contour inputs on every rank (contour.cpp, no exchange)
        fp = dco.compute_flow(mid_q, past_q, cfg)
        ff = dco.compute_flow(mid_q, future_q, cfg)
        mp = dco.gradient_amplitude(dco.flow_to_polar(*fp, with_theta=False)[0])
        mf = dco.gradient_amplitude(dco.flow_to_polar(*ff, with_theta=False)[0])
        m_fuse = dco.normalize_amplitude(dco.box_filter(dco.fuse_amplitudes(fp, ff, mp, mf, cfg), cfg.box_radius))
        edges, m_i = dco.extract_depth_contours_prefiltered(dco.gaussian_blur(mid_gray, cfg.gauss_sigma), m_fuse, cfg)
        qw = m_fuse.shape[1]
        self._mark("flow+contour")
        # stereo per band: only the vertical pass waits for the band above, and
        # its carry travels in chunks of slices, so band k+1's vertical pass of
        # chunk c overlaps band k's chunk c+1 (a pipeline, not a serial chain)
        sparse = {}
        nd = cfg.d_max - cfg.d_min + 1
        step = self.chunk or nd
        chunks = [(d0, min(nd, d0 + step)) for d0 in range(0, nd, step)]
        for k in sorted(self.plans):
            b = self.plans[k]
            dco.stereo_band_begin(mid_q[b.sub0:b.sub1].contiguous(), right_q[b.sub0:b.sub1].contiguous(), b, cfg,
                                  fw, fh)
            for d0, d1 in chunks:
                carry = None
                if b.carry_row > 0:
                    carry = L.get_carry((k, d0), torch.empty((d1 - d0, fw // 2), dtype=torch.float64, device="cuda"))
                carry_out = dco.stereo_band_vpass(b, cfg, fw, fh, d0, d1, carry)
                if carry_out is not None:
                    L.put_carry((k, d0), carry_out)
            _, sparse[k] = dco.stereo_band_end(b, cfg, fw, fh)
        self._mark("stereo")
        # frame-wide sparse mean from the bands' exact partials
        stats = {k: self._sparse_stats(sparse[k]) for k in self.plans}
        allstats = L.gather_stats(stats)
        mean, exact = self._combine(allstats)
        if not exact or self.force_sequential_mean:
            # outside the exactness guard the bands' partial sums may round
            # differently from the reference's row-major sum (densify.cpp:60-68):
            # gather the whole sparse map and take the sequential mean of it
            mean = self._sequential_mean(L.gather_rows(sparse))
        self._mean = mean
        # assembly of each band's rows (+ 2-row halo)
        systems, anchors, const = {}, {}, {}
        for k, b in self.plans.items():
            s0, s1 = self._sub(b)
            sub_sparse = torch.full((s1 - s0, fw), math.nan, dtype=torch.float32, device="cuda")
            sub_sparse[b.frow0 - s0:b.frow1 - s0] = sparse[k]
            pre = None
            if k in self.prev and cfg.lambda_s2 > 0.0:
                pre = torch.full((s1 - s0, fw), math.nan, dtype=torch.float32, device="cuda")
                pre[b.frow0 - s0:b.frow1 - s0] = self.prev[k]
            sys = dco.ConstraintSystem(fw, s1 - s0)
            anchors[k], const[k] = self._assemble(sub_sparse, edges[s0:s1], m_fuse[s0 // 2:], qw,
                                                  m_i[s0:s1], pre, b.frow0 - s0, b.frow1 - b.frow0, sys)
            systems[k] = (sys, b.frow0 - s0)
        tot = L.gather_stats({k: [float(anchors[k]), const[k], 0.0, 0.0] for k in self.plans})
        anchors_total = int(sum(t[0] for t in tot))
        const_total = sum(t[1] for t in tot)
        self._mark("assemble")
        # the solve over all bands
        dense = {}
        if anchors_total == 0:  # pipeline.cpp:236-242: keep the previous dense map
            for k, b in self.plans.items():
                dense[k] = self.prev.get(k, torch.full((b.frow1 - b.frow0, fw), math.nan, device="cuda"))
            unsolvable = True
        else:
            views = {k: dco.band_system(sys, r0, self.plans[k].frow1 - self.plans[k].frow0)
                     for k, (sys, r0) in systems.items()}
            if isinstance(L, LocalLinks):
                ks = sorted(self.plans)
                out, st = dco.band_solve_local([self.solvers[k] for k in ks], [views[k] for k in ks], cfg,
                                               anchors_total, const_total, history_cap=0)
                dense = dict(zip(ks, out))
                self.iterations = st[0].iterations
            else:
                for k in self.plans:
                    dense[k], st = self.solvers[k].solve(views[k], cfg, anchors_total, const_total, history_cap=0)
                    self.iterations = st.iterations
            unsolvable = False
        self._mark("solve")
        # composite of each band's rows
        res = {}
        for k, b in self.plans.items():
            r0, r1 = b.frow0, b.frow1
            vr = vrgb[r0:r1] if vrgb is not None else torch.zeros((r1 - r0, fw, 3), device="cuda")
            vd = vdepth[r0:r1] if vdepth is not None else torch.full((r1 - r0, fw), math.nan, device="cuda")
            comp, mask = dco.composite(mid_rgb[r0:r1].contiguous(), dense[k], vr.contiguous(), vd.contiguous())
            res[k] = dict(dense=dense[k], composite=comp, mask=mask, sparse=sparse[k], rows=(r0, r1),
                          unsolvable=unsolvable)
            self.prev[k] = dense[k]
        self._mark("composite")
        self._close_marks()
        return res

    @staticmethod
    def _sparse_stats(rows):
        import ctypes

        out = (ctypes.c_double * 4)()
        dco._call(dco._lib().dco_band_sparse_stats, dco._p(rows), rows.numel(), out)
        return list(out)

    @staticmethod
    def _sequential_mean(full):
        """sparse_mean (densify.cpp:60-68) of the whole map: dco_sparse_mean,
        whose device path sums in row-major order whenever the guard fails."""
        import ctypes

        full = full.contiguous()
        mean = ctypes.c_double()
        dco._call(dco._lib().dco_sparse_mean, dco._p(full), full.numel(), ctypes.byref(mean))
        return mean.value

    @staticmethod
    def _combine(allstats):
        import ctypes

        flat = (ctypes.c_double * (4 * len(allstats)))(*[v for s in allstats for v in s])
        mean, exact = ctypes.c_double(), ctypes.c_int()
        st = dco._lib().dco_band_sparse_mean(flat, len(allstats), ctypes.byref(mean), ctypes.byref(exact))
        if st != 0:
            raise UnsolvableFrameError("dco_band_sparse_mean failed")
        return mean.value, bool(exact.value)

    def _assemble(self, sparse, edges, m_fuse, qw, m_i, pre, own0, own_rows, sys):
        import ctypes

        w, h = self.fw, sparse.shape[0]
        qh = m_fuse.shape[0]
        cs = sys.c_struct()
        anchors, const = ctypes.c_uint64(), ctypes.c_double()
        dco._call(dco._lib().dco_band_assemble, dco._p(sparse), dco._p(edges.contiguous()), dco._p(m_fuse.contiguous()),
                  qw, qh, dco._p(m_i.contiguous()), dco._p(pre), w, h, own0, own_rows, ctypes.byref(self.cfg),
                  self._mean, ctypes.byref(cs), ctypes.byref(anchors), ctypes.byref(const))
        return anchors.value, const.value
