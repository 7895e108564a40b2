#!/usr/bin/env python
"""DCO hot-path benchmark (BASELINE.json metric: frames/sec at 1280x720, D=128).

A step is one composited frame of the full DCO path for one stream in steady
state (previous-dense chain active): stereo (cross windows, AD-census cost,
aggregation, WTA, histogram refinement, sparse depth) + bidirectional flow +
depth contours + assemble + PCG/MR densify + render + composite — the body of
run_pipeline (reference src/pipeline.cpp:183-258).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU. Under torchrun the ranks come from the environment; a
plain `python bench.py --gpus N` (N > 1) re-launches itself under
torch.distributed.run with N ranks. Every rank runs --streams independent
pipeline streams concurrently (own dco_ctx + CUDA stream each; frames shard
across streams and GPUs, no data-path collective: "scaling": "weak"). A step
is one frame on every stream. The timed region is bracketed by a barrier +
cuda.synchronize; the reported time is the max over ranks. L2 is flushed
(160 MiB memset; the L2 is 126 MB) before every frame inside the timed region.

`value` times frames whose u8 inputs are already in HBM. `e2e` times the same
steps through the host-buffer C-ABI (dco_stream_push_gray8_host): pinned u8
frames H2D, the pipeline, the composite/mask/dense D2H.

--impl reference runs the reference's own public frame loop, dco::run_pipeline
(pipeline.cpp:108-321, oracle/_ref built unmodified from /root/reference), on
one process per host core, each over its own PGM stream with per-frame poses
and the OBJ cube, timed by the reference's own StageTimings.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W, H, D = 1280, 720, 128
NQ, NF = (W // 2) * (H // 2), W * H
METRIC = "stereo frames/sec at 1280x720 D=128 (1/2/4/8 B200) vs CPU; HBM GB/s fraction"
STREAMS_PER_GPU = 8
# the workload, identical in both arms' lines (arm-specific details go under "arm")
CONFIG = {
    "workload": "DCO frame 1280x720 D=128 steady state (stereo+flow+contour+densify+render+composite)",
    "width": W, "height": H, "disparities": D,
    "frames": "synthetic stereo video (paper_2203_02300_b200.synth), independent streams, d_pre chain active",
    "virtual_layer": "cube mesh (0.3 m) rendered per frame under a per-frame pose",
    "l2": "GPU arm: flushed (160 MiB written, L2 is 126 MB) before every frame, inside the timed region",
    "parallelism": "frames shard as independent streams: 8 per GPU x N GPUs (GPU arm), one per host core "
                   "(reference arm); no data-path collective",
}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled every 5 ms during the timed region
    (NVML; nvidia-smi -lms 100 as the fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.sm = []
        self.mx = None
        self.reasons = set()
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self.stop.is_set():
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for n, b in self.REASONS.items():
                            if bits & b:
                                self.reasons.add(n)
                    except Exception:
                        pass
                    time.sleep(0.005)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if self.nvml:
            sm, mx, reasons = self.sm, self.mx, self.reasons
        else:
            sm, mx, reasons = [], None, set()
            for ln in self.lines:
                f = [x.strip() for x in ln.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    mx = float(f[2])
                except ValueError:
                    continue
                for n, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_procs(mem_per_proc=0.8e9):
    """All host threads, bounded by memory (~0.8 GB per reference process at
    1280x720 D=128)."""
    n = os.cpu_count() or 1
    try:
        import psutil

        n = max(1, min(n, int(psutil.virtual_memory().available / mem_per_proc)))
    except Exception:
        pass
    return n


def _ref_stream_worker(job, barrier, out_q):
    """One reference process: writes its stream as PGM frames + manifest (per
    frame poses) + OBJ cube + config, waits for every process, then runs the
    reference's dco::run_pipeline over it (oracle/_ref)."""
    try:
        from oracle import ref, refseq
        from paper_2203_02300_b200.config import Config
        from paper_2203_02300_b200.synth import StereoVideo

        seed, nframes, root, cfg_dict, keep = job
        vid = StereoVideo(W, H, seed=seed)
        frames = [vid.frame(i) for i in range(nframes)]
        paths = refseq.write_sequence(root, frames, poses=[frame_pose(i) for i in range(nframes)],
                                      mesh=cube_mesh(0.3), cfg=Config(**cfg_dict), keep_outputs=keep)
        ref.lib()
        barrier.wait()
        t0 = time.monotonic()
        res = ref.run_pipeline(*paths)
        out_q.put((seed, res, t0, time.monotonic(), paths[2]))
    except Exception as e:  # report, don't hide
        out_q.put((job[0], "error: %s" % e, 0.0, 0.0, None))


def run_reference_streams(seeds, nframes, cfg, keep_first=()):
    """P = len(seeds) concurrent reference processes, one stream each (its own
    keyframe window and d_pre chain over `nframes` frames). Returns per-seed
    (frames, t0, t1, out_dir) in seed order; frames as ref.run_pipeline."""
    import multiprocessing as mp
    import shutil
    import tempfile

    ctx = mp.get_context("fork")
    base = tempfile.mkdtemp(prefix="dco_refarm_")
    barrier, q = ctx.Barrier(len(seeds)), ctx.Queue()
    procs = []
    for k, sd in enumerate(seeds):
        job = (sd, nframes, os.path.join(base, "s%d" % sd), cfg.as_dict(), keep_first if k == 0 else ())
        pr = ctx.Process(target=_ref_stream_worker, args=(job, barrier, q))
        pr.start()
        procs.append(pr)
    got = {}
    for _ in seeds:
        sd, res, t0, t1, out = q.get()
        got[sd] = (res, t0, t1, out)
    for pr in procs:
        pr.join()
    bad = [str(v[0]) for v in got.values() if isinstance(v[0], str)]
    if bad:
        shutil.rmtree(base, ignore_errors=True)
        raise RuntimeError(bad[0])
    return [got[sd] for sd in seeds], base


def stage_table(frames_lists, reps_label):
    """The reference's 14-stage schema (pipeline.cpp:57-82) over the given
    frames: mean / min / max ms per stage and of the frame total."""
    from paper_2203_02300_b200 import report

    samples = [f["stages"] for fl in frames_lists for f in fl]
    totals = [f["total"] for fl in frames_lists for f in fl]
    rows = report.summarize(samples, totals)
    text = report.format_bench_report(len(samples), rows)
    return {r[0]: round(r[1], 3) for r in rows}, "%s\n%s" % (reps_label, text)


def run_reference(args, world, rank):
    """--impl reference: the reference's own frame loop dco::run_pipeline
    (oracle/_ref, built unmodified from /root/reference) on every host core,
    one stream per process, on this arm's config / metric. Each process runs
    2 + 1 + W + K frames: the window fill, the first composited frame (no
    d_pre), W warm-up and K timed steady frames; a step is one frame on every
    process. value = sum over processes of K / (sum of its timed frames'
    StageTimings totals)."""
    import shutil

    from paper_2203_02300_b200.config import Config
    from paper_2203_02300_b200.sharding import stream_seeds

    if rank != 0:
        return
    cfg = Config(d_max=D - 1)
    procs = min(cpu_procs(), 96)
    nframes = 3 + args.warmup + args.steps
    w0 = time.monotonic()
    runs, base = run_reference_streams(stream_seeds(0, procs), nframes, cfg)
    wall = time.monotonic() - w0
    shutil.rmtree(base, ignore_errors=True)
    timed = [res[1 + args.warmup: 1 + args.warmup + args.steps] for res, _, _, _ in runs]
    if any(len(t) != args.steps for t in timed):
        raise RuntimeError("reference run returned fewer composited frames than requested")
    per_proc_s = [sum(f["total"] for f in t) / 1000.0 for t in timed]
    value = sum(args.steps / s for s in per_proc_s)
    ms_step = 1000.0 * statistics.mean(per_proc_s) / args.steps
    iters = [f["iterations"] for t in timed for f in t]
    stages, text = stage_table(timed, "reference run_pipeline, %d processes x %d timed frames" % (procs, args.steps))
    print(text, file=sys.stderr)
    sample = ("%d concurrent reference processes (dco::run_pipeline, oracle/_ref), one stream each: %d frames "
              "(window fill + first frame + %d warm-up + %d timed steady frames); value from the reference's own "
              "StageTimings frame totals; whole run %.1f s wall" % (procs, nframes, args.warmup, args.steps, wall))
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "config": dict(CONFIG),
        "arm": {"processes": procs, "cpu_model": cpu_model(), "frames_per_step": procs,
                "densify_iterations_mean": statistics.mean(iters), "stage_ms": stages},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": procs, "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def algorithmic_bytes(span, iters):
    """SURVEY §8(d) per-unit figures x units per launch."""
    if span == "solve":
        return 104.0 * NF * max(iters, 1)
    if span == "aggregate":
        return 8.0 * NQ * D + 4.0 * NQ
    if span == "cost":
        return 28.0 * NQ + 4.0 * NQ * D
    if span == "wta":
        return 4.0 * NQ * D + 4.0 * NQ
    return None


def cube_mesh(side, color=(1.0, 0.55, 0.1)):
    """make_cube_mesh (occlude.cpp:89-105) centred at the origin."""
    import numpy as np

    r = np.float32(side) / np.float32(2.0)
    v = np.array([[r if i & 1 else -r, r if i & 2 else -r, r if i & 4 else -r] for i in range(8)], np.float32)
    faces = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    t = np.array([tri for f in faces for tri in ((f[0], f[1], f[2]), (f[0], f[2], f[3]))], np.int32)
    return v, t, np.tile(np.array(color, np.float32), (8, 1))


def frame_pose(k):
    """Per-frame manifest pose: the cube spinning 1.5 m in front of the camera."""
    import math

    a = 0.05 * k
    c, s = math.cos(a), math.sin(a)
    return [c, 0.0, s, 0.0, 0.0, 1.0, 0.0, 0.0, -s, 0.0, c, 1.5, 0.0, 0.0, 0.0, 1.0]


def run_ours(args, world, rank, local):
    import threading as th

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    from paper_2203_02300_b200 import dco, report
    from paper_2203_02300_b200.config import Config
    from paper_2203_02300_b200.sharding import Group, stream_seeds
    from paper_2203_02300_b200.synth import StereoVideo

    group = Group(world, local, "nccl")
    barrier = group.barrier

    S = args.streams
    cfg = Config(d_max=D - 1)
    nframes = 32
    vids = [StereoVideo(W, H, seed=sd) for sd in stream_seeds(rank, S)]
    host = [[v.frame(i) for i in range(nframes)] for v in vids]
    dev_l = [torch.from_numpy(np.stack([f[0] for f in h])).cuda() for h in host]
    dev_r = [torch.from_numpy(np.stack([f[1] for f in h])).cuda() for h in host]
    # virtual layer: the pipeline's cube mesh (make_cube_mesh, occlude.cpp:89-105)
    # rendered on the device every frame under a per-frame pose
    # (render_virtual + transform_mesh, pipeline.cpp:247-252)
    mesh_v, mesh_t, mesh_c = cube_mesh(0.3)

    tstreams = [torch.cuda.Stream() for _ in range(S)]
    streams = []
    for s in range(S):
        with torch.cuda.stream(tstreams[s]):
            st = dco.Stream(W, H, cfg, ctx=dco.new_context(tstreams[s]))
            st.set_mesh(mesh_v, mesh_t, mesh_c)
            streams.append(st)
    # > the 126 MB L2; written as int32 words (fill_ on a 4-byte view runs at ~6.6 TB/s, zero_ on
    # bytes at ~3.7: the same 160 MiB written, half the time)
    flush = [torch.empty(40 << 20, dtype=torch.int32, device="cuda") for _ in range(S)]
    pos = [0] * S

    def push(s, want=False):
        with torch.cuda.stream(tstreams[s]):
            streams[s].set_next_pose(frame_pose(pos[s]))
            flush[s].fill_(pos[s])  # L2 flush before every frame, inside the timed region
            r = streams[s].push_gray8(dev_l[s][pos[s] % nframes], dev_r[s][pos[s] % nframes], want_result=want)
        pos[s] += 1
        return r

    # fill each window (3 frames), reach the d_pre steady state, then W warm-ups
    for _ in range(3 + args.warmup):
        for s in range(S):
            push(s)
    torch.cuda.synchronize()
    launches0 = sum(st.launches() for st in streams)
    main = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0.record(main)
        for ts in tstreams:
            ts.wait_event(t0)
        for _ in range(args.steps):
            for s in range(S):
                push(s)
        for ts in tstreams:
            e = torch.cuda.Event()
            e.record(ts)
            main.wait_event(e)
        t1.record(main)
        torch.cuda.synchronize()
        barrier()
    total_ms = t0.elapsed_time(t1)
    launches = sum(st.launches() for st in streams) - launches0
    iters = push(0, want=True).densify_iterations

    # isolated per-span timing (one stream, nothing concurrent) for the roofline
    streams[0].set_timing(True)
    for _ in range(5):
        push(0)
    torch.cuda.synchronize()
    spans, nt = streams[0].span_times()
    streams[0].set_timing(False)

    # end to end through the host-buffer C-ABI: pinned u8 in, composite/mask/
    # dense out, S host threads (ctypes releases the GIL) driving S contexts
    hl = [[torch.from_numpy(f[0]).pin_memory() for f in h] for h in host]
    hr = [[torch.from_numpy(f[1]).pin_memory() for f in h] for h in host]
    # the frame's outputs as run_pipeline writes them (pipeline.cpp:266-268):
    # composite RGB bytes, mask bytes, dense floats
    outs = [(torch.empty((H, W, 3), dtype=torch.uint8).pin_memory(), torch.empty((H, W), dtype=torch.uint8).pin_memory(),
             torch.empty((H, W)).pin_memory()) for _ in range(S)]

    # S x K frames in total, handed out one at a time: a thread whose stream
    # runs ahead takes the next frame of its own stream (each stream's frames
    # stay in order, d_pre chained), so the run does not end on a tail of
    # stragglers while the other threads idle
    tickets = [0]
    lock = th.Lock()

    def e2e_worker(s):
        while True:
            with lock:
                if tickets[0] <= 0:
                    return
                tickets[0] -= 1
            k = pos[s] % nframes
            streams[s].set_next_pose(frame_pose(pos[s]))
            streams[s].push_gray8_host_encoded(hl[s][k], hr[s][k], *outs[s])
            pos[s] += 1

    def e2e_run(total):
        tickets[0] = total
        ths = [th.Thread(target=e2e_worker, args=(s,)) for s in range(S)]
        [t.start() for t in ths]
        [t.join() for t in ths]

    e2e_run(2 * S)
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e2e_run(args.steps * S)
    e2e_total = 1000.0 * (time.perf_counter() - w0)
    barrier()

    total_ms, e2e_total = group.max_over_ranks([total_ms, e2e_total], device="cuda")
    if rank != 0:
        for st in streams:
            st.close()
        group.close()
        return

    frames = world * S * args.steps
    value = frames / (total_ms / 1000.0)
    e2e_value = frames / (e2e_total / 1000.0)
    per_frame = {k: v / max(nt, 1) for k, v in spans.items()}
    dominant = max(per_frame, key=per_frame.get)
    peak, peak_src = peaks()
    ab = algorithmic_bytes(dominant, iters)
    roof = None
    if ab is not None:
        achieved = ab / (per_frame[dominant] / 1000.0) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(dominant)
        roof = {"kernel": dominant, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes": ab, "ms_per_launch": per_frame[dominant],
                "timing": "CUDA events around the span, one stream alone (5 frames)"}
        if dominant == "solve":
            roof["note"] = ("algorithmic bytes = SURVEY 8(d) 104 B per unknown per CG iteration (the reference's "
                            "per-iteration vector streams) x iterations; k_pcg_tmem keeps that state in registers, "
                            "TMEM and shared memory, so its DRAM traffic ('traffic') is a small fraction and frac > 1 "
                            "means faster than streaming the reference formulation at HBM peak. Its own bound is the "
                            "per-iteration grid barrier + SM issue (DESIGN.md section 4).")
    agg_ab = algorithmic_bytes("aggregate", 0)
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "config": dict(CONFIG),
        "arm": {"streams_per_gpu": S, "frames_per_step": S * world, "gpus": world,
                "stage_ms_reference_schema": dict(zip(report.STAGE_NAMES,
                                                      [round(x, 4) for x in report.stages_from_spans(spans, nt)]))},
        "roofline": roof,
        "aggregation_roofline": {"achieved": agg_ab / (per_frame["aggregate"] / 1000.0) / 1e9, "peak": peak,
                                 "unit": "GB/s", "frac": agg_ab / (per_frame["aggregate"] / 1000.0) / 1e9 / peak},
        "stage_ms": {k: round(v, 4) for k, v in per_frame.items()},
        "frame_ms_isolated": round(sum(per_frame.values()), 4),
        "densify_iterations": iters,
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": 2 * NF * S * world,
                "d2h_bytes_per_step": (NF * 3 + NF + NF * 4) * S * world,
                "path": "dco_stream_push_gray8_host_encoded (pinned host u8 in; out: the frame's files' contents "
                        "as run_pipeline writes them, pipeline.cpp:266-268 -- composite RGB bytes (write_ppm), "
                        "mask bytes (write_mask_pgm), dense floats (write_pfm))"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    for st in streams:
        st.close()
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as e:  # report, don't hide
            line["cpu_baseline"] = {"value": None, "error": str(e)[:300]}
    print(json.dumps(line))
    group.close()


def cpu_baseline(cfg):
    """The reference timed on this box's host cores on a bounded sample of the
    same workload: P concurrent processes, each the reference's own
    dco::run_pipeline over a 4-frame stream of the GPU arm's scene (window
    fill, a first composited frame, then one timed steady frame, d_pre chained
    by the reference itself). value = sum over processes of 1 / (its steady
    frame's StageTimings total).

    Parity on the same run: stream 0 (the GPU arm's stream-0 seed and poses)
    is pushed through a fresh GPU stream; both composited frames' dense maps
    (the reference's dense_NNNN.pfm) and CG iteration counts are compared."""
    import shutil

    import numpy as np
    import torch

    from oracle import refseq
    from paper_2203_02300_b200 import dco
    from paper_2203_02300_b200.sharding import stream_seeds
    from paper_2203_02300_b200.synth import StereoVideo

    procs = min(cpu_procs(), 96)
    seeds = stream_seeds(0, procs)
    nframes = 4
    w0 = time.monotonic()
    runs, base = run_reference_streams(seeds, nframes, cfg, keep_first=(1, 2))
    wall = time.monotonic() - w0
    steady = [res[1] for res, _, _, _ in runs]
    value = sum(1000.0 / f["total"] for f in steady)
    stages, text = stage_table([[f] for f in steady], "cpu_baseline: reference run_pipeline, steady frame x %d" % procs)
    print(text, file=sys.stderr)

    # GPU vs reference on stream 0
    res0, _, _, out0 = runs[0]
    vid = StereoVideo(W, H, seed=seeds[0])
    s = dco.Stream(W, H, cfg)
    v, t, c = cube_mesh(0.3)
    s.set_mesh(v, t, c)
    gpu_iters, max_abs = [], []
    for i in range(nframes):
        l8, r8 = vid.frame(i)
        s.set_next_pose(frame_pose(i))
        r = s.push_gray8(torch.from_numpy(l8).cuda(), torch.from_numpy(r8).cuda())
        if r.composited:
            torch.cuda.synchronize()
            dense = dco.view_tensor(s.views().dense, (H, W), torch.float32).cpu().numpy()
            want = refseq.read_pfm(os.path.join(out0, "dense_%04d.pfm" % (i - 1)))
            want = np.where(np.isinf(want), np.nan, want)
            gpu_iters.append(int(r.densify_iterations))
            max_abs.append(float(np.nanmax(np.abs(dense.astype(np.float64) - want))))
    s.close()
    shutil.rmtree(base, ignore_errors=True)
    return {"value": value, "unit": "frames/s", "cores": procs, "kind": "reference", "cpu_model": cpu_model(),
            "sample": "%d concurrent reference processes (dco::run_pipeline, oracle/_ref), one 4-frame stream each; "
                      "timed: each stream's steady frame (StageTimings total); run wall %.1f s" % (procs, wall),
            "stage_ms": stages,
            "parity_stream0": {"reference_iterations": [f["iterations"] for f in res0],
                               "gpu_iterations": gpu_iters, "dense_max_abs_m": max_abs,
                               "frames": "first composited (no d_pre) and steady"}}


def relaunch_under_torchrun(n):
    """`python bench.py --gpus N` without torchrun: re-exec with N ranks."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % n,
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=STREAMS_PER_GPU, help="concurrent pipeline streams per GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_under_torchrun(args.gpus)
    world, rank, local = dist_setup()
    if world != args.gpus:
        sys.exit("bench.py: --gpus %d but WORLD_SIZE=%d (launch one rank per GPU)" % (args.gpus, world))
    if args.impl == "ours":
        import torch

        if torch.cuda.device_count() < world:
            sys.exit("bench.py: --gpus %d but only %d visible GPUs" % (world, torch.cuda.device_count()))
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
