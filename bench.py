"""Benchmark of the B200 hot path: gather-pyramid filter fwd+bwd (BASELINE metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4a|c3|c2|c4b] [--no-e2e] [--no-cpu] [--no-also]

Default workload (BASELINE.json configs[4a], the metric's 1080p multi-GPU
config): 64 frames of 1920x1080, 3-level 5x5 pyramid, fp32, forward + backward
with parameter gradients, sharded by frame over N GPUs (64/N frames per GPU;
strong scaling, no collective on the data path).  Inputs are synthetic with the
BASELINE distributions (seeded): noisy radiance from the fused placement op at
0.25 spp over a log-normal bank with 1% x100 fireflies, albedo demodulation
U[0.05,1], N(0,1) logits and upstream gradient.  The working set (~50 GB at
N=1) is far larger than the 126 MB L2, so no explicit flush is needed.

One JSON line (rank 0).  `value` = device-timed Mpix/s over all ranks (max over
ranks of the CUDA-event time).  `roofline` = the dominant kernel (level-0
backward) timed live with CUDA events on its own stream; `step_roofline` =
SURVEY.md 8(d)'s fwd+bwd algorithmic bytes per step over the step time.
`e2e` = same metric through the host-buffer path (pinned H2D of every input,
D2H of every result, copies inside the timed region).  `cpu_baseline` /
`--impl reference` = the reference algorithm (oracle port, numpy float64) on
the host cores.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (frames_total, H, W, L, k, logit dtype, description)
    "c4a": (64, 1080, 1920, 3, 5, "f32",
            "c4a: 64 x 1920x1080 frames, 3-level 5x5 pyramid, fp32 logits+radiance, fwd+bwd "
            "(logit, radiance and demod grads), sharded by frame"),
    "c3": (1, 2160, 3840, 4, 7, "bf16",
           "c3: 1 x 3840x2160, 4-level 7x7 pyramid, bf16 logits, fp32 radiance/accumulate, fwd+bwd"),
    "c2": (64, 256, 256, 4, 5, "f32",
           "c2: 64 x 256x256 crops, 4-level 5x5 pyramid, fp32, fwd+bwd"),
    "c4b": (1, 4320, 7680, 4, 7, "f32",
            "c4b: one 7680x4320 frame, 4-level 7x7 pyramid, fp32, forward only; N>1 splits it into "
            "row bands with a one-round NVLink halo exchange (bands.py)"),
}
FWD_ONLY = {"c4b"}
# per-worker samples of each workload for the reference arm (H, W, L, k, with
# backward): a 960x540 crop at the workload's pyramid depth and kernel size
# (c2: one of its 256^2 frames; c4b: forward only, like the workload)
CPU_SAMPLES = {"c4a": (540, 960, 3, 5, True), "c3": (540, 960, 4, 7, True), "c2": (256, 256, 4, 5, True),
               "c4b": (540, 960, 4, 7, False)}


# ---------------------------------------------------------------------------
# algorithmic bytes


def level_shapes(h, w, L):
    s = [(h, w)]
    while len(s) < L:
        s.append(((s[-1][0] + 1) // 2, (s[-1][1] + 1) // 2))
    return s


def logit_channels(l, L, k):
    return k * k + (4 if l < L - 1 else 0)


def algorithmic_bytes(h, w, L, k, sl, sg, channels=3):
    """(FWD, BWD, dominant-kernel) bytes per frame.  FWD/BWD follow 8(d):
    each pass reads its inputs and writes its outputs once, intermediates
    excluded.  Dominant kernel = level-0 backward: logits0 read, g_logits0
    write, upstream/noisy/demod/out read, g_noisy/g_demod written."""
    img = 4 * channels
    dims = level_shapes(h, w, L)
    n0 = h * w
    lg = sum(a * b * logit_channels(l, L, k) for l, (a, b) in enumerate(dims))
    fwd = n0 * 3 * img + lg * sl
    bwd = n0 * 6 * img + lg * (sl + sg)
    dom = n0 * (logit_channels(0, L, k) * (sl + sg) + 6 * img)
    return fwd, bwd, dom


# ---------------------------------------------------------------------------
# CPU legs: the reference algorithm (oracle port, float64) on host cores


def _cpu_worker(arg):
    seed, (h, w, L, k, bwd) = arg
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np

    from oracle import pyramid as op
    rng = np.random.default_rng(seed)
    logits = op.random_logits(h, w, L, k, rng, temporal=True)
    noisy = rng.lognormal(-1.0, 1.5, (h, w, 3)) * (rng.uniform(size=(h, w, 1)) < 0.25)
    demod = rng.uniform(0.05, 1.0, (h, w, 3))
    up = rng.normal(size=(h, w, 3))
    t0 = time.perf_counter()
    out, tape = op.forward(noisy, logits, None, demod, k=k)
    if bwd:
        op.backward(tape, up)
    return time.perf_counter() - t0


def cpu_pool_size(sample=None):
    h, w, L, k, _ = sample or CPU_SAMPLES["c4a"]
    cores = len(os.sched_getaffinity(0))
    try:
        import psutil
        ram = psutil.virtual_memory().available
    except Exception:
        ram = 8 << 30
    # measured ~1.7 GB RSS for one 960x540 L3 k5 fwd+bwd; scales with pixels
    # and logit channels
    per_proc = 2.2 * (1 << 30) * (h * w) / (540 * 960) * (2 * k * k + 4) / 54
    return max(1, min(cores, int(ram // per_proc)))


class CpuPool:
    def __init__(self, procs):
        self.procs = procs
        ctx = mp.get_context("spawn")
        env_threads = os.environ.get("OMP_NUM_THREADS")
        os.environ["OMP_NUM_THREADS"] = "1"
        self.pool = ctx.Pool(procs)
        if env_threads is None:
            os.environ.pop("OMP_NUM_THREADS", None)
        else:
            os.environ["OMP_NUM_THREADS"] = env_threads

    def step(self, seed, sample):
        t0 = time.perf_counter()
        self.pool.map(_cpu_worker, [(seed * 1000 + i, sample) for i in range(self.procs)])
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample_desc(procs, workload="c4a"):
    h, w, L, k, bwd = CPU_SAMPLES[workload]
    return (f"{procs} worker processes x one {w}x{h} L{L} k{k} {'fwd+bwd' if bwd else 'fwd'} (float64 "
            f"numpy oracle port of the reference, OMP_NUM_THREADS=1 each) per step; CPU {cpu_model()}")


def run_cpu(steps, warmup, workload="c4a"):
    sample = CPU_SAMPLES[workload]
    procs = cpu_pool_size(sample)
    pool = CpuPool(procs)
    try:
        for i in range(warmup):
            pool.step(100 + i, sample)
        times = [pool.step(i, sample) for i in range(steps)]
    finally:
        pool.close()
    h, w = sample[0], sample[1]
    t = sum(times) / len(times)
    return {"value": procs * h * w / t / 1e6, "procs": procs, "sec_per_step": t}


# ---------------------------------------------------------------------------
# GPU arm


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def synthetic_inputs(B, H, W, L, k, ldt, device, seed):
    """BASELINE distributions: density softplus(GRF sigma=8) standardised,
    0.25 spp placement over a log-normal(-1, 1.5) bank with 1% x100
    fireflies (fused placement op), albedo U[0.05,1], N(0,1) logits."""
    import torch
    import torch.nn.functional as F

    from paper_2602_08642_b200 import ops
    g = torch.Generator(device=device).manual_seed(seed)
    noisy = torch.empty(B, 3, H, W, device=device)
    sig = 8.0
    r = int(3 * sig)
    xs = torch.arange(-r, r + 1, device=device, dtype=torch.float32)
    ker = torch.exp(-xs ** 2 / (2 * sig * sig))
    ker = ker / ker.sum()
    S = 2
    for b in range(B):
        z = torch.randn(1, 1, H, W, generator=g, device=device)
        z = F.conv2d(F.pad(z, (r, r, 0, 0), mode="circular"), ker.view(1, 1, 1, -1))
        z = F.conv2d(F.pad(z, (0, 0, r, r), mode="circular"), ker.view(1, 1, -1, 1))
        z = (z - z.mean()) / z.std()
        scores = torch.log(F.softplus(z))[0].contiguous()
        bank = torch.exp(-1.0 + 1.5 * torch.randn(1, S, 3, H, W, generator=g, device=device))
        fire = torch.rand(1, S, 1, H, W, generator=g, device=device) < 0.01
        bank = torch.where(fire, bank * 100.0, bank).contiguous()
        ops.place_fused(scores, bank, 0.25, seed=seed, frame0=b, noisy=noisy[b:b + 1])
        del z, scores, bank, fire
    demod = torch.rand(B, 3, H, W, generator=g, device=device) * 0.95 + 0.05
    ltype = {"f32": torch.float32, "bf16": torch.bfloat16}[ldt]
    logits = [torch.randn(B, logit_channels(l, L, k), h, w, generator=g, device=device).to(ltype)
              for l, (h, w) in enumerate(level_shapes(H, W, L))]
    up = torch.randn(B, 3, H, W, generator=g, device=device)
    return noisy, demod, logits, up


class Runner:
    """Pre-allocated fwd+bwd through the C ABI (no per-step allocation)."""

    def __init__(self, noisy, demod, logits, up, k):
        import torch

        from paper_2602_08642_b200 import _lib, ops
        self.lib = _lib.load()
        self.check = _lib.check
        self.noisy, self.demod, self.logits, self.up = noisy, demod, logits, up
        self.desc = ops._desc(noisy, logits, demod, None, k, "native")
        tb, wb = C.c_size_t(), C.c_size_t()
        self.check(self.lib.ssb_pyr_tape_bytes(C.byref(self.desc), C.byref(tb)), "tape")
        self.check(self.lib.ssb_pyr_workspace_bytes(C.byref(self.desc), C.byref(wb)), "ws")
        dev = noisy.device
        self.tape = torch.empty(max(tb.value, 1), dtype=torch.uint8, device=dev)
        self.ws = torch.empty(max(wb.value, 1), dtype=torch.uint8, device=dev)
        self.out = torch.empty_like(noisy)
        self.g_noisy = torch.empty_like(noisy)
        self.g_demod = torch.empty_like(noisy)
        self.g_logits = [torch.empty_like(z) for z in logits]
        self.fio = _lib.PyrFwdIO()
        self.fio.noisy, self.fio.demod, self.fio.out = noisy.data_ptr(), demod.data_ptr(), self.out.data_ptr()
        self.bio = _lib.PyrBwdIO()
        self.bio.noisy, self.bio.demod = noisy.data_ptr(), demod.data_ptr()
        self.bio.out, self.bio.upstream = self.out.data_ptr(), up.data_ptr()
        self.bio.g_noisy, self.bio.g_demod = self.g_noisy.data_ptr(), self.g_demod.data_ptr()
        for l, (z, gz) in enumerate(zip(logits, self.g_logits)):
            self.fio.logits[l] = z.data_ptr()
            self.bio.logits[l] = z.data_ptr()
            self.bio.g_logits[l] = gz.data_ptr()
        self.tape_p = C.c_void_p(self.tape.data_ptr())
        self.ws_p = C.c_void_p(self.ws.data_ptr())

    fwd_only = False

    def step(self, stream):
        s = C.c_void_p(stream)
        rc = self.lib.ssb_pyr_forward(C.byref(self.desc), C.byref(self.fio), self.tape_p, s)
        if rc:
            self.check(rc, "ssb_pyr_forward")
        if self.fwd_only:
            return
        rc = self.lib.ssb_pyr_backward(C.byref(self.desc), C.byref(self.bio), self.tape_p, self.ws_p, s)
        if rc:
            self.check(rc, "ssb_pyr_backward")


class BandRunner:
    """c4b at N > 1: this rank owns one row band of the frame (bands.py):
    halo rows of each pooled level and one Lhat row per level move over peer
    memory (CUDA IPC + P2P stores + generation flags; no NCCL on the data
    path), every level runs the library's level kernel on the band's
    row-extended buffers."""

    fwd_only = True

    def __init__(self, dist, rank, world, H, W, L, k, dev):
        import torch

        from paper_2602_08642_b200 import bands
        self.bands = bands
        pl = bands.plan(H, L, k, world)
        self.eng = bands.BandForward(pl, rank, H, W, L, k, bands.CudaCompute(k), device=dev)
        g = torch.Generator(device=dev).manual_seed(77 + rank)
        self.eng.noisy_own.copy_(torch.rand(self.eng.noisy_own.shape, generator=g, device=dev))
        self.eng.demod_own.copy_(torch.rand(self.eng.demod_own.shape, generator=g, device=dev) * 0.95 + 0.05)
        for z in self.eng.logits_own:
            z.copy_(torch.randn(z.shape, generator=g, device=dev))
        self.tr = bands.PeerTransport(dist, self.eng, dev)
        self.tr.setup()

    def step(self, stream):
        self.eng.run(self.tr)


def chain_order():
    """The library's level-0-last backward (float32, 3 channels, demodulated,
    no history, L >= 2; csrc/pyr_chain.cuh) -- every bench workload uses it
    unless SSB_NO_CHAIN / SSB_NO_TMA disable it."""
    return os.environ.get("SSB_NO_CHAIN") != "1" and os.environ.get("SSB_NO_TMA") != "1"


def launches_per_step(L, fwd_only=False):
    # forward: (L-1) pooling + L level kernels
    names = [f"pool{l}->{l + 1}" for l in range(L - 1)]
    names += [f"fwd_l{l}" for l in range(L - 1, -1, -1)]
    if fwd_only:
        return names
    if chain_order():
        # backward, level 0 last: upsample-transpose pre-pass, levels 1..L-1,
        # the level-1 pool chain (L >= 3), level 0 (final outputs)
        names += ["bwd_up"] + [f"bwd_l{l}" for l in range(1, L)]
        names += (["bwd_chain"] if L >= 3 else []) + ["bwd_l0"]
    else:
        # backward: L level kernels (fine -> coarse) + the coarse -> fine sweep
        names += [f"bwd_l{l}" for l in range(L)] + ["bwd_final"]
    return names


def time_device(runner, steps, warmup, L, dist, world):
    import torch
    lib = runner.lib
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    for _ in range(warmup):
        runner.step(sp)
    torch.cuda.synchronize()
    names = launches_per_step(L, runner.fwd_only)
    per = len(names)
    cap = per * steps
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * cap)]
    for e in evs:  # torch creates the underlying cudaEvent lazily, on first record
        e.record(stream)
    ev_arr = (C.c_void_p * (2 * cap))(*[e.cuda_event for e in evs])
    count = C.c_int(0)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n0 = lib.ssb_launch_count()
    lib.ssb_set_launch_events(ev_arr, cap, C.byref(count))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        runner.step(sp)
    t1.record(stream)
    lib.ssb_set_launch_events(None, 0, None)
    torch.cuda.synchronize()
    launches = lib.ssb_launch_count() - n0
    ms = t0.elapsed_time(t1)
    if dist:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = tt.item()
        dist.barrier()
    durs = {nm: [] for nm in names}
    for i in range(count.value):
        durs[names[i % per]].append(evs[2 * i].elapsed_time(evs[2 * i + 1]))
    mean = {nm: (sum(v) / len(v) if v else None) for nm, v in durs.items()}
    return ms / steps, mean, launches


def time_e2e(dev, frames, steps, k, H, W, L, ldt, chunk=4, pool_frames=16):
    """Host-buffer path: per frame chunk, H2D of noisy/demod/logits/upstream
    from pinned memory, fwd+bwd, D2H of out/g_logits/g_noisy/g_demod.  Copies
    run on their own streams and overlap compute of the neighbouring chunk."""
    import torch

    chunk = max(1, min(chunk, frames))
    pool_frames = max(chunk, min(pool_frames, frames))
    pool_frames -= pool_frames % chunk
    lt = torch.float32 if ldt == "f32" else torch.bfloat16
    lvl = level_shapes(H, W, L)

    def host(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True)

    h_in = {"noisy": host((pool_frames, 3, H, W), torch.float32),
            "demod": host((pool_frames, 3, H, W), torch.float32),
            "up": host((pool_frames, 3, H, W), torch.float32)}
    h_lg = [host((pool_frames, logit_channels(l, L, k), h, w), lt) for l, (h, w) in enumerate(lvl)]
    h_out = {n: host((pool_frames, 3, H, W), torch.float32) for n in ("out", "g_noisy", "g_demod")}
    h_glg = [host((pool_frames, logit_channels(l, L, k), h, w), lt) for l, (h, w) in enumerate(lvl)]
    for t in list(h_in.values()) + h_lg:
        t.uniform_(0.05, 1.0)
    # NBUF device chunk buffers: the H2D of chunk i + NBUF waits only for the
    # D2H of chunk i (3 measured no better than 2)
    NBUF = 2
    bufs = []
    for _ in range(NBUF):
        d_n = torch.empty(chunk, 3, H, W, device=dev)
        d_d = torch.empty_like(d_n)
        d_u = torch.empty_like(d_n)
        d_lg = [torch.empty(chunk, logit_channels(l, L, k), h, w, device=dev, dtype=lt)
                for l, (h, w) in enumerate(lvl)]
        r = Runner(d_n, d_d, d_lg, d_u, k)
        bufs.append(r)
    s_h2d, s_comp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    in_bytes = sum(t[0:1].numel() * t.element_size() for t in list(h_in.values()) + h_lg) * frames
    out_bytes = sum(t[0:1].numel() * t.element_size() for t in list(h_out.values()) + h_glg) * frames

    def one_step():
        ev_h2d = [torch.cuda.Event() for _ in range(NBUF)]
        ev_comp = [torch.cuda.Event() for _ in range(NBUF)]
        ev_d2h = [None] * NBUF
        for ci, f0 in enumerate(range(0, frames, chunk)):
            r = bufs[ci % NBUF]
            p0 = f0 % pool_frames
            sl = slice(p0, p0 + chunk)
            with torch.cuda.stream(s_h2d):
                if ev_d2h[ci % NBUF] is not None:
                    s_h2d.wait_event(ev_d2h[ci % NBUF])
                r.noisy.copy_(h_in["noisy"][sl], non_blocking=True)
                r.demod.copy_(h_in["demod"][sl], non_blocking=True)
                r.up.copy_(h_in["up"][sl], non_blocking=True)
                for z, hz in zip(r.logits, h_lg):
                    z.copy_(hz[sl], non_blocking=True)
                ev_h2d[ci % NBUF].record(s_h2d)
            s_comp.wait_event(ev_h2d[ci % NBUF])
            r.step(s_comp.cuda_stream)
            ev_comp[ci % NBUF].record(s_comp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_comp[ci % NBUF])
                h_out["out"][sl].copy_(r.out, non_blocking=True)
                h_out["g_noisy"][sl].copy_(r.g_noisy, non_blocking=True)
                h_out["g_demod"][sl].copy_(r.g_demod, non_blocking=True)
                for hz, gz in zip(h_glg, r.g_logits):
                    hz[sl].copy_(gz, non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_d2h)
                ev_d2h[ci % NBUF] = e
        torch.cuda.synchronize()

    one_step()
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    dt = (time.perf_counter() - t0) / steps
    return dt, in_bytes, out_bytes


def time_e2e_compat(frames=2, H=1080, W=1920, L=3, k=5):
    """The drop-in caller's cost: the reference's own call
    shapes through compat (reconstruct_core + reconstruct_backward on HWC
    float64 numpy arrays, the reference KernelField layout with the 25-logit
    temporal group at level 0), float32 kernels; wall clock per frame,
    including the host<->device transfers of every float64 input and result
    and the device-side HWC <-> planar transposes."""
    import time

    import numpy as np
    import torch

    from paper_2602_08642_b200 import compat
    rng = np.random.default_rng(5)
    shapes = level_shapes(H, W, L)
    chans = [k * k + 4 + k * k] + [k * k + 4] * (L - 2) + [k * k]

    class KF:  # the reference KernelField's shape (pyramid.py:56-68)
        def __init__(self, logits):
            self.logits = logits
    kf = KF([rng.normal(0, 1, (h, w, c)) for (h, w), c in zip(shapes, chans)])
    noisy = rng.lognormal(-1.0, 1.5, (H, W, 3))
    demod = rng.uniform(0.05, 1.0, (H, W, 3))
    up = rng.normal(size=(H, W, 3))
    prev = compat.precision()
    compat.set_precision("f32")
    try:
        def frame():
            out, tape = compat.pyramid.reconstruct_core(noisy, kf, None, demod)
            g = compat.pyramid.reconstruct_backward(tape, up)
            return out, g
        frame()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(frames):
            frame()
        dt = (time.perf_counter() - t0) / frames
    finally:
        compat.set_precision(prev)
    h2d = 8 * (3 * H * W * 3 + sum(h * w * c for (h, w), c in zip(shapes, chans)))
    d2h = 8 * (3 * H * W * 3 + sum(h * w * c for (h, w), c in zip(shapes, chans)))
    return {"value": round(H * W / dt / 1e6, 3), "unit": "Mpix/s", "ms_per_frame": round(dt * 1e3, 2),
            "h2d_bytes_per_frame": h2d, "d2h_bytes_per_frame": d2h,
            "path": "compat.reconstruct_core + reconstruct_backward (the reference's call shapes: HWC float64 "
                    "numpy in and out, level-0 logits with the temporal group), float32 kernels, one 1080p "
                    "L3 k5 frame per call, wall clock"}


def pcie_gbs(dev, nbytes=1 << 30):
    """Pinned host <-> device copy bandwidth of this box: one 1 GiB copy each
    way, then both at once on two streams (aggregate), after a warm-up -- the
    ceiling of the e2e number."""
    import torch
    h, h2 = (torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2))
    d, d2 = (torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2))
    out = []
    for src, dst in ((h, d), (d, h)):  # best of 3 (one-off hiccups)
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out.append(best)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    bidir = 0.0
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        bidir = max(bidir, 2 * nbytes / (time.perf_counter() - t0) / 1e9)
    out.append(bidir)
    del h, h2, d, d2
    return out


def gpu_arm(args, rank, world, local_rank, dist):
    import torch
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    frames_total, H, W, L, k, ldt, desc = WORKLOADS[args.workload]
    if frames_total % world and frames_total > 1:
        raise SystemExit(f"{frames_total} frames do not split over {world} GPUs")
    B = max(1, frames_total // world)
    fwd_only = args.workload in FWD_ONLY
    if fwd_only and world > 1:
        runner = BandRunner(dist, rank, world, H, W, L, k, dev)
    else:
        noisy, demod, logits, up = synthetic_inputs(B, H, W, L, k, ldt, dev, seed=1234 + rank)
        runner = Runner(noisy, demod, logits, up, k)
        runner.fwd_only = fwd_only
    sampler = ClockSampler(local_rank)
    sampler.start()
    ms, kern, launches = time_device(runner, args.steps, args.warmup, L, dist, world)
    clocks = sampler.stop()
    sl = 2 if ldt == "bf16" else 4
    fwd_b, bwd_b, dom_b = algorithmic_bytes(H, W, L, k, sl, sl)
    px_total = H * W if fwd_only else B * world * H * W
    value = px_total / (ms * 1e-3) / 1e6
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    if fwd_only:
        lg0 = logit_channels(0, L, k) * sl
        dom_name, dom_b = "fwd_l0", H * W * (lg0 + 36) // (world if world > 1 else 1)
        step_bytes = fwd_b
    else:
        dom_name, step_bytes = "bwd_l0", fwd_b + bwd_b
    dom_ms = kern.get(dom_name)
    # DRAM traffic of the dominant kernel from the committed ncu capture
    # (tools/ncu_traffic.py -> profiles/ncu_traffic.json), per launch like `achieved`
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        ent = tr.get(args.workload, {}).get(dom_name)
        if ent:
            traffic = int(ent["bytes_per_frame"] * B)
    except (OSError, ValueError, KeyError):
        pass
    dom_gbs = dom_b * B / (dom_ms * 1e-3) / 1e9 if dom_ms else None
    # per-GPU step bytes: c4b at N > 1 splits ONE frame into N row bands, so
    # each rank moves ~1/N of the frame's bytes (band halos are not algorithmic)
    if fwd_only and world > 1:
        step_bytes = step_bytes / world
    step_gbs = step_bytes * B / (ms * 1e-3) / 1e9
    res = {
        "metric": f"pyramidal filter {'fwd' if fwd_only else 'fwd+bwd'} throughput ({args.workload})",
        "value": round(value, 3),
        "unit": "Mpix/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong" if frames_total > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32" if ldt == "f32" else "f32 (bf16 logits)",
        "data": "synthetic, BASELINE config distributions (seeded); no dataset",
        "config": {"workload": desc, "frames_total": frames_total * (1 if frames_total > 1 else world),
                   "frames_per_gpu": B, "height": H, "width": W, "levels": L, "ksize": k,
                   "logit_dtype": ldt, "parallelism": f"frame-sharded x{world}, no collective",
                   "l2": "working set >> 126 MB L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "kernel": "bwd_l0 (level-0 backward: softmax recompute, "
                     "logit grads, gather-transpose, final g_noisy/g_demod)" if not fwd_only else
                     "fwd_l0 (level-0 forward: softmax, k x k gather, upsample, remod)",
                     "achieved": round(dom_gbs, 1) if dom_gbs else None, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(dom_gbs / peak, 4) if dom_gbs else None, "traffic": traffic,
                     "algorithmic_bytes_per_launch": dom_b * B,
                     "ms_per_launch": round(dom_ms, 4) if dom_ms else None,
                     "share_of_step": round(dom_ms / ms, 3) if dom_ms else None},
        "step_roofline": {"achieved": round(step_gbs, 1), "peak": peak, "unit": "GB/s",
                          "frac": round(step_gbs / peak, 4),
                          "bytes_per_frame": {"fwd": fwd_b, "bwd": 0 if fwd_only else bwd_b}},
        "step_dram": None if fwd_only else step_dram(args.workload, value / max(world, 1), peak),
        "kernels_ms": {kk: (round(v, 4) if v else None) for kk, v in kern.items()},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    return res, runner


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4a")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-also", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        frames_total, H, W, L, k, ldt, desc = WORKLOADS[args.workload]
        # the reference CPU path is float64 numpy; bounded samples per step
        steps = args.steps
        warm = min(args.warmup, 1)
        r = run_cpu(steps, warm, args.workload)
        fwd_only = args.workload in FWD_ONLY
        res = {"impl": "reference",
               "metric": f"pyramidal filter {'fwd' if fwd_only else 'fwd+bwd'} throughput ({args.workload})",
               "value": round(r["value"], 4), "unit": "Mpix/s", "n_gpus": world, "steps": steps,
               "warmup": warm, "ms_per_step": round(r["sec_per_step"] * 1e3, 1),
               "higher_is_better": True, "scaling": "strong" if frames_total > 1 else "weak",
               "vs_baseline": None,
               "dtype": "f64", "data": "synthetic, BASELINE config distributions (seeded)",
               "config": {"workload": desc, "sample": cpu_sample_desc(r["procs"], args.workload)},
               "cpu_baseline": {"value": round(r["value"], 4), "unit": "Mpix/s",
                                "cores": r["procs"], "kind": "port",
                                "sample": cpu_sample_desc(r["procs"], args.workload)},
               "e2e": {"value": round(r["value"], 4), "unit": "Mpix/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(res), flush=True)
        return

    dist = None
    if world > 1:
        import torch.distributed as tdist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        tdist.init_process_group("nccl")
        dist = tdist
    res, runner = gpu_arm(args, rank, world, local_rank, dist)
    frames_total, H, W, L, k, ldt, _ = WORKLOADS[args.workload]

    # e2e through the host-buffer path
    if not args.no_e2e and args.workload not in FWD_ONLY:
        B = max(1, frames_total // world)
        del runner
        import torch
        torch.cuda.empty_cache()
        dt, ib, ob = time_e2e(torch.device("cuda", local_rank), B, max(1, min(args.steps, 3)),
                              k, H, W, L, ldt)
        if dist:
            tt = torch.tensor([dt], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = tt.item()
        h2d, d2h, bidir = pcie_gbs(torch.device("cuda", local_rank))
        # copies overlap each other and the compute: the PCIe ceiling is the
        # step's bytes at the measured aggregate (both directions at once) rate
        ceil = B * H * W / max((ib + ob) / (bidir * 1e9), ib / (h2d * 1e9), ob / (d2h * 1e9)) / 1e6
        res["e2e"] = {"value": round(B * world * H * W / dt / 1e6, 3), "unit": "Mpix/s",
                      "h2d_bytes_per_step": ib * world, "d2h_bytes_per_step": ob * world,
                      "path": "ops C-ABI from pinned host buffers, chunked H2D/compute/D2H overlap",
                      "pcie_gbs_measured": {"h2d": round(h2d, 1), "d2h": round(d2h, 1),
                                            "both_directions": round(bidir, 1)},
                      "pcie_ceiling_mpix_s": round(ceil * world, 3),
                      "frac_of_pcie_ceiling": round(B * H * W / dt / 1e6 / ceil, 4)}
    else:
        res["e2e"] = None
    if rank == 0 and world == 1 and not args.no_e2e and args.workload == "c4a":
        res["e2e_compat"] = time_e2e_compat()

    if rank == 0 and world == 1 and not args.no_cpu:
        r = run_cpu(1, 1, args.workload)  # (one warm-up step: worker imports out of the timing)
        res["cpu_baseline"] = {"value": round(r["value"], 4), "unit": "Mpix/s", "cores": r["procs"],
                               "kind": "port", "sample": cpu_sample_desc(r["procs"], args.workload)}
    if rank == 0 and world == 1 and not args.no_also and args.workload == "c4a":
        res["also"] = also_measurements()
    if rank == 0:
        print(json.dumps(res), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def step_dram(workload, mpix_s, peak):
    """Achieved DRAM bandwidth of the whole step: the DRAM bytes per pixel
    that ncu measured for every kernel of one step of this workload
    (tools/gpu_step_traffic.sh -> profiles/step_traffic.json; cold,
    serialized launches) times the live pixel rate.  Supplementary to the
    algorithmic-bytes step_roofline (which counts only the minimum bytes)."""
    try:
        ent = json.load(open(os.path.join(ROOT, "profiles", "step_traffic.json")))[workload]
    except (OSError, ValueError, KeyError):
        return None
    gbs = ent["dram_bytes_per_px"] * mpix_s / 1e3
    return {"dram_bytes_per_px": ent["dram_bytes_per_px"], "achieved": round(gbs, 1), "peak": peak,
            "unit": "GB/s", "frac": round(gbs / peak, 4), "source": ent.get("source", "")}


def also_measurements():
    """The other BASELINE configs on the same box: c3 (4K, L4, k7, bf16
    logits), c4b (8K fwd), and the 8(f) rows (temporal warp, score gradient)."""
    import torch
    out = {}
    frames, H, W, L, k, ldt, desc = WORKLOADS["c3"]
    noisy, demod, logits, up = synthetic_inputs(1, H, W, L, k, ldt, torch.device("cuda"), seed=99)
    r = Runner(noisy, demod, logits, up, k)
    ms, kern, _ = time_device(r, 20, 3, L, None, 1)
    fwd_b, bwd_b, dom_b = algorithmic_bytes(H, W, L, k, 2, 2)
    peak = 6556.8
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    out["c3"] = {"workload": desc, "mpix_s": round(H * W / (ms * 1e-3) / 1e6, 2),
                 "ms_per_step": round(ms, 4),
                 "step_frac_of_hbm": round((fwd_b + bwd_b) / (ms * 1e-3) / 1e9 / peak, 4),
                 "bwd_l0_frac_of_hbm": round(dom_b / (kern["bwd_l0"] * 1e-3) / 1e9 / peak, 4),
                 "step_dram": step_dram("c3", H * W / (ms * 1e-3) / 1e6, peak),
                 "kernels_ms": {kk: (round(v, 4) if v else None) for kk, v in kern.items()}}
    del noisy, demod, logits, up, r
    torch.cuda.empty_cache()
    frames, H, W, L, k, ldt, desc = WORKLOADS["c4b"]
    noisy, demod, logits, up = synthetic_inputs(1, H, W, L, k, ldt, torch.device("cuda"), seed=98)
    r = Runner(noisy, demod, logits, up, k)
    r.fwd_only = True
    ms, kern, _ = time_device(r, 20, 3, L, None, 1)
    fwd_b, _, _ = algorithmic_bytes(H, W, L, k, 4, 4)
    out["c4b"] = {"workload": desc + " (N=1: full frame)", "mpix_s": round(H * W / (ms * 1e-3) / 1e6, 2),
                  "ms_per_frame": round(ms, 4),
                  "fwd_frac_of_hbm": round(fwd_b / (ms * 1e-3) / 1e9 / peak, 4),
                  "kernels_ms": {kk: (round(v, 4) if v else None) for kk, v in kern.items()}}
    del noisy, demod, logits, up, r
    torch.cuda.empty_cache()
    out.update(small_configs(peak))
    out.update(call_shapes(peak))
    out.update(next_rows(peak))
    return out


def call_shapes(peak, frames=4, H=1080, W=1920, L=3, k=5):
    """The reference's other call shapes of the filter, fwd+bwd
    at 4 x 1080p L3 k5 fp32: frame 1 of optimize.evaluate_step (the 25-tap
    temporal group over the warped history, optimize.py:209), reconstruct_core's
    default demod=None, and C = 12 batched draws (optimize.py:433-437).  Bytes
    per 8(d) with the history terms (prev read in fwd, prev + g_prev in bwd,
    k*k more level-0 logits)."""
    import torch

    from paper_2602_08642_b200 import ops
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(11)
    shapes = level_shapes(H, W, L)
    out = {}
    for name, C, hist, dem in (("history", 3, True, True), ("no_demod", 3, False, False), ("draws_c12", 12, False, True)):
        noisy = torch.rand(frames, C, H, W, generator=g, device=dev)
        demod = (torch.rand(frames, C, H, W, generator=g, device=dev) * 0.95 + 0.05) if dem else None
        prev = torch.rand(frames, C, H, W, generator=g, device=dev) if hist else None
        logits = [torch.randn(frames, ops.logit_channels(l, L, k, has_prev=hist and l == 0), h, w, generator=g,
                              device=dev) for l, (h, w) in enumerate(shapes)]
        up = torch.randn(frames, C, H, W, generator=g, device=dev)

        # the batched draws' backward takes no parameter gradients
        # (optimize.py:467: reconstruct_backward(..., want_param_grads=False))
        want = name != "draws_c12"

        def step():
            o, t = ops.pyramid_forward(noisy, logits, demod, prev, ksize=k)
            ops.pyramid_backward(t, up, want_param_grads=want)
        ms = _time_cuda(step, steps=10, warmup=3)
        img = 4 * C
        lg = sum(a * b * ops.logit_channels(l, L, k, has_prev=hist and l == 0) for l, (a, b) in enumerate(shapes))
        n0 = H * W
        fwd = n0 * img * ((3 if dem else 2) + (1 if hist else 0)) + lg * 4
        if want:
            bwd = n0 * img * ((6 if dem else 4) + (2 if hist else 0)) + lg * 8
        else:  # logits, upstream, demod in; g_noisy out
            bwd = n0 * img * (3 if dem else 2) + lg * 4
        out[f"shape_{name}"] = {
            "workload": f"{frames} x 1920x1080 L3 k5 fp32 fwd+bwd, " + {
                "history": "with the temporal group over a warped history (evaluate_step frame 1)",
                "no_demod": "demod=None (reconstruct_core's default)",
                "draws_c12": "C = 12 (4 batched draws sharing the kernels), no parameter gradients "
                             "(optimize.py:467)"}[name],
            "mpix_s": round(frames * n0 / (ms * 1e-3) / 1e6, 1), "ms_per_step": round(ms, 4),
            "frac_of_hbm": round(frames * (fwd + bwd) / (ms * 1e-3) / 1e9 / peak, 4)}
        del noisy, demod, prev, logits, up
        torch.cuda.empty_cache()
    return out


def small_configs(peak):
    """The remaining BASELINE configs: c2 (64 x 256^2, L4 k5 fp32 fwd+bwd) as
    throughput; c1 (one 1080p frame: fused placement + demod + L3 k5 forward)
    and c0 (one 256^2 frame, the same pipeline; L2-resident) as per-frame
    latency of a CUDA-graph replay of the whole inference path."""
    import torch
    import torch.nn.functional as F

    from paper_2602_08642_b200 import ops
    out = {}
    frames, H, W, L, k, ldt, desc = WORKLOADS["c2"]
    noisy, demod, logits, up = synthetic_inputs(frames, H, W, L, k, ldt, torch.device("cuda"), seed=97)
    r = Runner(noisy, demod, logits, up, k)
    ms, kern, _ = time_device(r, 20, 3, L, None, 1)
    fwd_b, bwd_b, dom_b = algorithmic_bytes(H, W, L, k, 4, 4)
    out["c2"] = {"workload": desc, "mpix_s": round(frames * H * W / (ms * 1e-3) / 1e6, 1),
                 "ms_per_step": round(ms, 4),
                 "step_frac_of_hbm": round(frames * (fwd_b + bwd_b) / (ms * 1e-3) / 1e9 / peak, 4),
                 "kernels_ms": {kk: (round(v, 4) if v else None) for kk, v in kern.items()}}
    del noisy, demod, logits, up, r
    out.update(latency_configs(peak))
    return out


def latency_configs(peak):
    """c1 / c0: per-frame latency of a CUDA-graph replay of the inference path
    (fused placement + demod + L3 k5 forward), with the placement alone timed
    the same way; plus the fused training placement (relaxed, with the
    density gradient) at 8 x 1080p as a throughput line."""
    import ctypes as C

    import torch
    import torch.nn.functional as F

    from paper_2602_08642_b200 import ops
    out = {}
    for name, H, W in (("c1", 1080, 1920), ("c0", 256, 256)):
        L, k = 3, 5
        dev = torch.device("cuda")
        g = torch.Generator(device=dev).manual_seed(7)
        z = torch.randn(1, 1, H, W, generator=g, device=dev)
        ker = torch.exp(-torch.arange(-24, 25, device=dev, dtype=torch.float32) ** 2 / 128.0)
        ker = ker / ker.sum()
        z = F.conv2d(F.pad(z, (24, 24, 0, 0), mode="circular"), ker.view(1, 1, 1, -1))
        z = F.conv2d(F.pad(z, (0, 0, 24, 24), mode="circular"), ker.view(1, 1, -1, 1))
        scores = torch.log(F.softplus((z - z.mean()) / z.std()))[0].contiguous()
        bank = torch.exp(-1.0 + 1.5 * torch.randn(1, 2, 3, H, W, generator=g, device=dev))
        bank = torch.where(torch.rand(1, 2, 1, H, W, generator=g, device=dev) < 0.01, bank * 100, bank).contiguous()
        demod = torch.rand(1, 3, H, W, generator=g, device=dev) * 0.95 + 0.05
        logits = [torch.randn(1, logit_channels(l, L, k), h, w, generator=g, device=dev)
                  for l, (h, w) in enumerate(level_shapes(H, W, L))]
        noisy = torch.empty(1, 3, H, W, device=dev)
        wsb = C.c_size_t()
        ops._lib.load().ssb_density_workspace_bytes(1, H, W, C.byref(wsb))
        ws = torch.empty(wsb.value, dtype=torch.uint8, device=dev)
        outb = torch.empty_like(noisy)

        iws = None
        if H * W <= (1 << 20):
            iwb = C.c_size_t()
            ops._lib.load().ssb_infer_small_workspace_bytes(1, H, W, L, C.byref(iwb))
            iws = torch.empty(iwb.value, dtype=torch.uint8, device=dev)

        def infer():
            # the library's inference path (ops.infer): one cooperative kernel
            # for small frames (c0), placement + pyramid_forward otherwise (c1)
            if iws is not None:
                ops.infer(scores, bank, demod, logits, 0.25, ksize=k, seed=3, noisy=noisy, out=outb, workspace=iws)
            else:
                ops.place_fused(scores, bank, 0.25, seed=3, noisy=noisy, workspace=ws)
                ops.pyramid_forward(noisy, logits, demod, ksize=k, out=outb)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                infer()
        torch.cuda.current_stream().wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            infer()
        reps = 200
        ms = _time_cuda(graph.replay, steps=reps, warmup=10)
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            ops.place_fused(scores, bank, 0.25, seed=3, noisy=noisy, workspace=ws)
        ms_p = _time_cuda(g2.replay, steps=reps, warmup=10)
        fwd_b, _, _ = algorithmic_bytes(H, W, L, k, 4, 4)
        out[name] = {"workload": f"{name}: one {W}x{H} frame, fused placement (0.25 spp) + demod + "
                                 f"3-level 5x5 forward, fp32, CUDA-graph replay",
                     "us_per_frame": round(ms * 1e3, 2),
                     "placement_us": round(ms_p * 1e3, 2),
                     "mpix_s": round(H * W / (ms * 1e-3) / 1e6, 1),
                     "fwd_frac_of_hbm": round((fwd_b + 19 * H * W) / (ms * 1e-3) / 1e9 / peak, 4),
                     "placement_frac_of_hbm": round(19 * H * W / (ms_p * 1e-3) / 1e9 / peak, 4)}
        del graph, g2, scores, bank, demod, logits, noisy, outb
    # fused training placement: relaxed estimator + density gradient, 8 x 1080p
    B, H, W = 8, 1080, 1920
    g = torch.Generator(device="cuda").manual_seed(5)
    scores = torch.randn(B, H, W, generator=g, device="cuda") * 0.5
    bank = torch.exp(-1.0 + 1.5 * torch.randn(B, 2, 3, H, W, generator=g, device="cuda"))
    noisy = torch.empty(B, 3, H, W, device="cuda")
    wsb = C.c_size_t()
    ops._lib.load().ssb_density_workspace_bytes(B, H, W, C.byref(wsb))
    ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
    res = {}
    res["r"] = ops.place(scores, bank, 0.25, "relaxed", noisy=noisy, want_grad=True, workspace=ws)
    gbuf = res["r"]["grad"]

    def train_place():
        ops.place(scores, bank, 0.25, "relaxed", noisy=noisy, want_grad=True, workspace=ws)
    ms = _time_cuda(train_place, steps=20, warmup=3)
    # scores 4 + samples read 12 E[n] (3 at 0.25 spp) + noisy 12 + grad 12
    out["place_train"] = {"workload": "8 x 1920x1080, fused placement, relaxed estimator + density gradient "
                                      "(the training default), fp32 out, float64 decisions",
                          "mpix_s": round(B * H * W / (ms * 1e-3) / 1e6, 1), "ms": round(ms, 4),
                          "frac_of_hbm": round(31 * B * H * W / (ms * 1e-3) / 1e9 / peak, 4)}
    del scores, bank, noisy, ws, gbuf, res
    torch.cuda.empty_cache()
    return out


def _time_cuda(fn, steps=20, warmup=3):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def next_rows(peak):
    """SURVEY.md 8(f) rows measured on the same box: the temporal warp and its
    transpose (8 x 1080p, fp32, |motion| <= 2 px) and the estimator backward to
    the density scores (8 x 1080p, fp32, 2 frames, sigma 1.5).  Algorithmic
    bytes: warp 36 B/px (prev, motion, out, validity), transpose 32 B/px
    (grad_out, motion, grad_prev), score grad 56 B/px (2 frames of g_input and
    grad_density, scores, g_scores)."""
    import torch

    from paper_2602_08642_b200 import ops
    B, H, W = 8, 1080, 1920
    n = B * H * W
    gen = torch.Generator(device="cuda").manual_seed(5)
    dev = torch.device("cuda")
    prev = torch.rand((B, 3, H, W), device=dev, generator=gen)
    motion = (torch.rand((B, 2, H, W), device=dev, generator=gen) - 0.5) * 4
    g = torch.randn((B, 3, H, W), device=dev, generator=gen)
    ms_w = _time_cuda(lambda: ops.warp(prev, motion))
    ms_b = _time_cuda(lambda: ops.warp_backward(g, motion))
    out = {"temporal_warp": {
        "workload": "8 x 1920x1080 fp32, 3 channels, motion U(-2, 2) px",
        "warp_mpix_s": round(n / (ms_w * 1e-3) / 1e6, 1), "warp_ms": round(ms_w, 4),
        "warp_frac_of_hbm": round(36 * n / (ms_w * 1e-3) / 1e9 / peak, 4),
        "transpose_mpix_s": round(n / (ms_b * 1e-3) / 1e6, 1), "transpose_ms": round(ms_b, 4),
        "transpose_frac_of_hbm": round(32 * n / (ms_b * 1e-3) / 1e9 / peak, 4)}}
    del prev, motion, g
    sc = torch.randn((B, H, W), device=dev, generator=gen)
    gi = torch.randn((B, 2, 3, H, W), device=dev, generator=gen)
    gd = torch.randn((B, 2, 3, H, W), device=dev, generator=gen)
    ms_s = _time_cuda(lambda: ops.score_grad(sc, gi, gd, 0.25, 1.5))
    out["score_grad"] = {
        "workload": "8 x 1920x1080 fp32 (float64 reductions), 2 frames, blur sigma 1.5",
        "mpix_s": round(n / (ms_s * 1e-3) / 1e6, 1), "ms": round(ms_s, 4),
        "frac_of_hbm": round(56 * n / (ms_s * 1e-3) / 1e9 / peak, 4)}
    del sc, gi, gd
    # tonemap + loss epilogue of one training step (8(f) row 4): tonemap of the
    # frame, losses + gradients against a reference with a warped history,
    # tonemap backward -- one fused kernel (ops.loss_epilogue).  Algorithmic
    # bytes = the epilogue's inputs and outputs: radiance, ref, ldr0_w, ref_w
    # (4 x 12) + validity, mask (2 x 4) + grad_radiance, g_ldr0_w (2 x 12) =
    # 80 B/px.  The three-launch composition (tonemap, losses, tonemap
    # backward: 152 B/px moved, intermediates partly L2-resident) is timed
    # beside it.
    rad = torch.rand((B, 3, H, W), device=dev, generator=gen) * 4
    ref = torch.rand((B, 3, H, W), device=dev, generator=gen)
    l0w = torch.rand((B, 3, H, W), device=dev, generator=gen)
    rw = torch.rand((B, 3, H, W), device=dev, generator=gen)
    val = (torch.rand((B, H, W), device=dev, generator=gen) > 0.1).float()
    msk = torch.ones((B, H, W), device=dev)
    tmo = (0.0, 1.0, 1.0, 0.5, 0.5)

    def composed():
        ldr = ops.tonemap(rad, tmo)
        r = ops.losses(ldr, ref, l0w, rw, validity=val, mask=msk, want_maps=False, want_grads=True)
        return ops.tonemap_backward(rad, tmo, r["g_ldr1"])
    ms_c = _time_cuda(composed)
    ms_e = _time_cuda(lambda: ops.loss_epilogue(rad, ref, tmo, l0w, rw, validity=val, mask=msk))
    out["loss_epilogue"] = {
        "workload": "8 x 1920x1080 fp32: tonemap, masked spatial + temporal losses with gradients, tonemap "
                    "backward, one fused kernel",
        "mpix_s": round(n / (ms_e * 1e-3) / 1e6, 1), "ms": round(ms_e, 4),
        "frac_of_hbm": round(80 * n / (ms_e * 1e-3) / 1e9 / peak, 4),
        "composed_3_launches_ms": round(ms_c, 4)}
    del rad, ref, l0w, rw, val, msk
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
