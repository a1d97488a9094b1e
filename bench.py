#!/usr/bin/env python
"""bench.py -- CS-frame Gpixels/s of the fused residual + block-measurement encoder on B200.

Default workload (BASELINE.json configs[3], the config the metric's target is quoted on):
1080p 1920x1080 uint8, 240 frames, GOP 8, 16x16 blocks, M swept over {16,32,64,128}.  One
"step" = the whole hot path over that sequence for every M of the sweep (4 kernel launches,
one per measurement matrix), inputs resident in HBM.  value = CS pixels encoded / second
(key frames pass through and are not counted), whole job (all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C4]

Multi-GPU: `--gpus N` (N > 1) re-runs itself under torch.distributed.run with N ranks (or run it under
torchrun directly); every rank encodes its own independent sequence (weak scaling; GOPs are
independent, P:87 / SPEC.md:406) -- no data-path collective; a barrier and a MAX all-reduce of the
device time are the only communication.

--impl reference times the fp64 CPU oracle (oracle/, the slow correctness reference) on a
bounded sample of the same workload; on N>1 only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

L2_BYTES = 126 * 1024 * 1024


OUTPUTS = {"f32": None, "q16frame": 0, "q16row": 1}   # --output -> cs_encode_batch_q16 granularity


def alg_bytes(cfg, M, n_seq, output="f32"):
    """Algorithmic HBM bytes of one step for one M: every frame read once + every measurement
    written once: fp32 (4 B), or int16 codes (2 B) + fp32 scales
    (one per CS frame, or per CS frame and block row) for the f1 outputs."""
    nbx, nby = -(-cfg.W // cfg.B), -(-cfg.H // cfg.B)
    n_cs = cfg.T - -(-cfg.T // cfg.G)
    if output == "f32":
        return n_seq * (cfg.T * cfg.W * cfg.H + n_cs * nbx * nby * M * 4)
    n_scales = n_cs * (nby if output == "q16row" else 1)   # q16frame: one per CS frame
    return n_seq * (cfg.T * cfg.W * cfg.H + n_cs * nbx * nby * M * 2 + 4 * n_scales)


def cs_pixels(cfg, n_seq):
    return n_seq * (cfg.T - -(-cfg.T // cfg.G)) * cfg.W * cfg.H


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.period = period_s

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_traffic(workload):
    """Per-launch DRAM bytes from the committed ncu --set full summary (profiles/), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(workload)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------ ours
def timed_steps(args, launch, n_launch, stream, dev, world, flush=None):
    """W untimed warm-up steps, then K timed steps of n_launch launches each between ONE CUDA-event pair on the
    launching stream (barrier + synchronize on both sides, clocks sampled during the region, device time = max
    over ranks), then -- after a 0.5 s pause -- a per-launch attribution pass: min(K, 20) steps with an event
    pair around every launch.  With an L2 flush before every launch there is one pass of K steps, timed by the
    launches' pairs.  Returns (ms_total, launch_ms[i] = the pair times of launch i, clk)."""
    import torch
    import torch.distributed as dist

    def step(ev=None):
        for i in range(n_launch):
            if flush is not None:   # L2 flush outside the launch's event pair (inputs smaller than L2)
                flush.fill_(1)
            if ev is not None:
                ev[i][0].record(stream)
            launch(i)
            if ev is not None:
                ev[i][1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    K = args.steps
    Kp = K if flush is not None else min(K, 20)   # steps of the per-launch-event pass
    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in range(n_launch)]
           for _ in range(Kp)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # The timed region: K steps queued back to back, one event pair around them.  (An event record between
    # two kernels keeps the second one's prologue from overlapping the first one's tail -- the K1 kernels are
    # launched with programmatic dependent launch -- so the per-launch events live in a pass of their own below.
    # Inputs smaller than L2 are flushed before every launch, which needs the per-launch events: one pass.)
    with ClockSampler(dev.index or 0) as clk:
        t0.record(stream)
        for k in range(K):
            step(evs[k] if flush is not None else None)
        t1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_total = t0.elapsed_time(t1)
    if flush is None:   # per-launch attribution pass (an event pair around every launch), after the timed region
        time.sleep(0.5)   # and after a pause: sustained load lowers the throughput, and the
        for k in range(Kp):   # attribution should see the launches as the first steps of the region did
            step(evs[k])
        torch.cuda.synchronize(dev)
    launch_ms = [[evs[k][i][0].elapsed_time(evs[k][i][1]) for k in range(Kp)] for i in range(n_launch)]
    if flush is not None:   # the step time excludes the flushes: sum of the launches' own event times (Kp == K)
        ms_total = sum(sum(col) for col in launch_ms)
    if world > 1:
        tt = torch.tensor([ms_total], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total = float(tt.item())
    return ms_total, launch_ms, clk


def l2_clean_times(launch, n_launch, stream, dev, reps):
    """Per-launch device time with L2 holding only CLEAN lines before each launch: a read-only pass
    over a buffer 4x the L2 (a reduction) evicts whatever the previous launch left -- including its
    dirty output tail, whose write-back would otherwise be charged to the next launch -- without
    leaving dirty lines itself.  Outside the timed region; for the per-M attribution only."""
    import torch
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    buf = torch.ones(4 * l2 // 4, dtype=torch.int32, device=dev)
    out = []
    for i in range(n_launch):
        evs = []
        for _ in range(reps):
            buf.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launch(i)
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize(dev)
        out.append(sum(a.elapsed_time(b) for a, b in evs) / reps)
    del buf
    return out


def timed_output_parity(cfg, Ms, phis, frames_h, results, gran, n_samples=400, seed=0):
    """Oracle check of the outputs the timed steps wrote (every step rewrites the same outputs, so the
    buffers after timing are the timed results): n_samples (CS frame, block) entries of the rank's
    first stream per M, each recomputed one by one from the definition (oracle.measure_entries).
    fp32: |y_gpu - y| <= 1e-5 * S (S = 0 -> exactly 0).  q16: the dequantised code is within half a
    quantisation step (plus the tolerance band) of the exact y."""
    import oracle
    rng = np.random.default_rng(seed)
    nbx, nby = -(-cfg.W // cfg.B), -(-cfg.H // cfg.B)
    nblk = nbx * nby
    n_cs_s = cfg.T - -(-cfg.T // cfg.G)
    worst, n_bad, n = 0.0, 0, 0
    for M, phi, res in zip(Ms, phis, results):
        ci = rng.integers(0, n_cs_s, size=n_samples)
        bi = rng.integers(0, nblk, size=n_samples)
        bi[: min(n_samples, 8)] = nblk - 1 - np.arange(min(n_samples, 8))   # always include the ragged last blocks
        y, S = oracle.measure_entries(frames_h[0], phi, cfg.G, cfg.B, ci, bi)
        if gran is None:
            g = res.view(-1, nblk, M)[ci, bi].double().cpu().numpy()
            d = np.abs(g - y)
            bad = (d > 1e-5 * S) | ((S == 0) & (g != 0))
            with np.errstate(divide="ignore", invalid="ignore"):
                rel = np.where(S > 0, d / np.where(S > 0, S, 1.0), 0.0)
        else:
            codes, scales = res
            c = codes.view(-1, nblk, M)[ci, bi].double().cpu().numpy()
            sc = scales.view(-1, nby)[ci, bi // nbx] if gran == 1 else scales.view(-1)[ci]
            sc = sc.double().cpu().numpy()[:, None]
            d = np.abs(c * sc - y)
            lim = sc * (0.5 + 2.0 ** -21) + 1e-5 * S + 2.0 ** -22 * np.abs(y)
            bad = d > lim
            rel = d / lim
        n_bad += int(bad.sum())
        n += y.size
        worst = max(worst, float(rel.max()))
    key = "max_rel" if gran is None else "max_err_over_bound"
    return {"entries": n_samples * len(Ms), "values": n, "n_bad": n_bad, key: worst, "ok": n_bad == 0,
            "how": f"{n_samples} sampled (CS frame, block) entries x M of the timed outputs vs oracle.measure_entries"}


def run_ours(args, cfg, Ms):
    import torch
    import torch.distributed as dist
    import paper_1311_1419_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    n_seq = cfg.S
    # rank r encodes its own independent streams (weak scaling)
    frames_h = synth.gen_video(cfg, streams=range(rank * n_seq, (rank + 1) * n_seq))
    frames = torch.from_numpy(frames_h).to(dev)
    encs, outs, qouts = [], [], []
    gran = OUTPUTS[args.output]
    for M in Ms:
        phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
        e = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
        encs.append(e)
        outs.append(torch.empty(e.out_shape(n_seq, cfg.T), dtype=torch.float32, device=dev))
        if gran is not None:
            qouts.append((torch.empty(e.out_shape(n_seq, cfg.T), dtype=torch.int16, device=dev),
                          torch.empty(e.q16_scale_shape(n_seq, cfg.T, gran), dtype=torch.float32, device=dev)))
    if gran is not None:
        outs = [None] * len(Ms)   # the q16 step does not touch the fp32 buffers; free them
        torch.cuda.empty_cache()
    stream = torch.cuda.current_stream(dev)
    if args.gop_phis:   # f4 variant: Phi(seed ^ g) per GOP index
        n_g = -(-cfg.T // cfg.G)
        for M, e in zip(Ms, encs):
            e.set_gop_phis([synth.phi_from_seed(synth.phi_seed() ^ g, M, cfg.B ** 2) for g in range(n_g)])
    # plan choice: the fastest of the planner's top plans (outputs are bit-identical across plans);
    # --tune-file reuses earlier choices (e.g. under ncu, so no tuning launches are profiled)
    tuned = {}
    if args.tune_file and os.path.exists(args.tune_file):
        with open(args.tune_file) as f:
            tuned = json.load(f)
    for i, e in enumerate(encs):
        key = f"{args.workload}:{Ms[i]}"
        if key in tuned:
            e.set_candidate(int(tuned[key]))
        elif not args.no_autotune and gran is None:
            e.autotune(frames, outs[i], max_candidates=args.tune_candidates, reps=2, stream=stream)
            tuned[key] = e.tuned_index()
        elif not args.no_autotune:
            # q16 outputs: time the planner's top plans on the q16 call itself (the epilogue differs,
            # so the fp32-tuned plan is not necessarily the fastest); codes are bitwise plan-independent
            best, best_ms = None, float("inf")
            for k in range(min(args.tune_candidates, e.num_candidates())):
                e.set_candidate(k)
                try:
                    e.encode_batch_q16(frames, gran, qouts[i][0], qouts[i][1], stream)   # warm-up
                except P.CSError:   # e.g. row scales need <= 40 block rows per tile: skip this plan
                    continue
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record(stream)
                for _ in range(2):
                    e.encode_batch_q16(frames, gran, qouts[i][0], qouts[i][1], stream)
                t1.record(stream)
                t1.synchronize()
                if t0.elapsed_time(t1) < best_ms:
                    best, best_ms = k, t0.elapsed_time(t1)
            if best is None:
                raise SystemExit(f"--output {args.output}: no candidate plan of M={Ms[i]} supports this output")
            e.set_candidate(best)
            tuned[key] = best
    if args.tune_file and rank == 0:
        with open(args.tune_file, "w") as f:
            json.dump(tuned, f)

    closed = args.op == "closed_loop"
    if not closed and os.environ.get("BENCH_STABLE_INPUTS", "1") != "0":   # the frames are resident before the timed region and nothing writes them: loads may overlap
        for e in encs:   # the previous launch's tail (cs_encoder_set_stable_inputs)
            e.set_stable_inputs(True)
    if closed:   # f4: key codec once per step (keys do not depend on M), then every M against them
        qsteps = P.key_qsteps(args.key_scale)
        keys, coef = encs[0].key_codec(frames, qsteps, stream=stream)

    # L2 between iterations (contract: flush it, or use inputs larger than it):
    #  * inputs >= 2 x L2 (C4, C5): nothing to do;
    #  * inputs < 2 x L2 but >= 2 x L2 / 11 (C3, C2), fp32 open-loop encode: the steps ROTATE over n_rot copies of the frames and
    #    n_rot output buffers (n_rot x input >= 2 x L2 + input), so a launch never finds its frames in L2 and the
    #    previous launches' dirty output is written back inside the region -- a stream of new data, no flush
    #    (back-to-back launches on ONE copy re-read 6% of the input from L2 and leave 36 of the 43 MB output
    #    dirty in L2: ncu --cache-control none; --no-rotate times that config with flushes instead);
    #  * smaller inputs (C1), or other ops / outputs below 2 x L2: L2 flushed before every launch, outside
    #    its event pair.
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    n_rot = 1
    if (frames.numel() < 2 * l2_bytes and gran is None and args.op == "encode" and not args.gop_phis
            and not args.no_rotate):
        n_rot = -(-2 * l2_bytes // frames.numel()) + 1
        if n_rot > 12:   # tiny inputs (C1): that many copies still fit in L2 together -- flush instead
            n_rot = 1
    frames_r = [frames] + [frames.clone() for _ in range(n_rot - 1)]
    outs_r = [[o] + [torch.empty_like(o) for _ in range(n_rot - 1)] for o in outs] if gran is None else None
    rot = [0]

    def launch(i, st=None):
        st = stream if st is None else st
        if closed:
            if i == 0:
                encs[0].key_codec(frames, qsteps, keys=keys, coef=coef, stream=st)
                return
            i -= 1
        e = encs[i]
        if closed:
            e.encode_batch_keys(frames, keys, outs[i], st)
        elif gran is None:
            if i == 0:
                rot[0] = (rot[0] + 1) % n_rot
            e.encode_batch(frames_r[rot[0]], outs_r[i][rot[0]], st)
        else:
            e.encode_batch_q16(frames, gran, qouts[i][0], qouts[i][1], st)

    small = frames.numel() < 2 * l2_bytes and n_rot == 1
    flush = torch.empty(4 * l2_bytes, dtype=torch.uint8, device=dev) if small else None
    ms_total, launch_ms, clk = timed_steps(args, launch, len(Ms) + (1 if closed else 0), stream, dev, world, flush)
    K = args.steps
    # per-launch attribution with a clean L2 before every launch (outside the timed region)
    clean_ms = l2_clean_times(launch, len(Ms) + (1 if closed else 0), stream, dev, max(3, min(K, 10)))
    if closed:
        clean_ms = clean_ms[1:]
    key_ms = None
    if closed:
        key_ms = statistics.mean(launch_ms[0])
        launch_ms = launch_ms[1:]

    # ---- end to end through the public host-buffer C-ABI call (copies inside the timed region)
    e2e = None
    if closed:
        e2e = {"value": None, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "how": "not measured: the closed loop has a device-buffer C-ABI call only"}
    elif not args.no_e2e:
        pin_in = torch.from_numpy(frames_h).pin_memory()
        if gran is None:
            pin_out = [torch.empty(e.out_shape(n_seq, cfg.T), dtype=torch.float32).pin_memory() for e in encs]

            def host_call():   # one public call per step: every M over the same host frames
                P.encode_batch_host_multi(encs, pin_in, pin_out)
            d2h = sum(o.numel() * 4 for o in pin_out)
            how = "cs_encode_batch_host_multi"
        else:
            pin_out = [(torch.empty(e.out_shape(n_seq, cfg.T), dtype=torch.int16).pin_memory(),
                        torch.empty(e.q16_scale_shape(n_seq, cfg.T, gran), dtype=torch.float32).pin_memory())
                       for e in encs]

            def host_call():
                P.encode_batch_host_multi_q16(encs, pin_in, gran, pin_out)
            d2h = sum(c.numel() * 2 + sc.numel() * 4 for c, sc in pin_out)
            how = "cs_encode_batch_host_multi_q16 (int16 codes + fp32 scales copied back)"
        host_call()   # warm-up (workspace allocation)
        e2e_steps = max(1, min(args.e2e_steps, K))
        if world > 1:
            dist.barrier()
        w0 = time.perf_counter()
        for _ in range(e2e_steps):
            host_call()
        w = (time.perf_counter() - w0) / e2e_steps
        if world > 1:
            tt = torch.tensor([w], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            w = float(tt.item())
        h2d = frames_h.nbytes                       # frames cross PCIe once per step
        e2e = {"value": world * len(Ms) * cs_pixels(cfg, n_seq) / w / 1e9, "unit": "Gpixel/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": w * 1e3,
               "how": how + " (all M encoders over the same pinned host frames: frames copied in once, H2D + "
                            "encodes + D2H pipelined in stream groups), wall clock around the synchronous C-ABI call"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    peak, peak_src = load_peaks()
    per_m = {}
    tot_bytes, tot_ms = 0.0, 0.0
    for i, M in enumerate(Ms):
        med = statistics.median(launch_ms[i])
        avg = statistics.mean(launch_ms[i])
        b = alg_bytes(cfg, M, n_seq, args.output)
        per_m[str(M)] = {"ms_median": med, "ms_mean": avg, "ms_mean_l2clean": clean_ms[i],
                         "frac_of_peak_l2clean": alg_bytes(cfg, M, n_seq, args.output) / (clean_ms[i] * 1e-3) / 1e9 / peak,
                         "gpix_s": cs_pixels(cfg, n_seq) / (avg * 1e-3) / 1e9,
                         "alg_gbs": b / (avg * 1e-3) / 1e9, "frac_of_peak": b / (avg * 1e-3) / 1e9 / peak,
                         "alg_bytes": b, "plan": encs[i].plan()}
        tot_bytes += b
        tot_ms += avg
    ms_step = ms_total / K
    # roofline: the step's algorithmic bytes over the step's time in the timed region (= bytes per launch over
    # the average launch duration there).  With L2 flushes between launches (small inputs) or the key-codec
    # launch in the step (closed loop) the K1 launches' own event pairs are the time base instead.
    achieved_pairs = tot_bytes / (tot_ms * 1e-3) / 1e9
    achieved = achieved_pairs if (small or closed) else tot_bytes / (ms_step * 1e-3) / 1e9
    # the committed ncu capture is of the default fp32 open-loop encode; other variants report null
    plain = args.output == "f32" and not closed and not args.gop_phis
    traffic = load_traffic(args.workload) if plain else None
    value = world * len(Ms) * cs_pixels(cfg, n_seq) / (ms_step * 1e-3) / 1e9
    in_mb = cfg.T * cfg.W * cfg.H * n_seq / 2 ** 20
    line = {
        "metric": "CS-frame Gpixels/s encoded (residual vs GOP key + block measurement Y = Phi R)",
        "value": value, "unit": "Gpixel/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8 in, fp16 x fp16 -> fp32 (tensor core kind::f16)", "data": "synthetic (seeded surveillance-like video, synth/)",
        "config": {"workload": args.workload, "W": cfg.W, "H": cfg.H, "T": cfg.T, "streams_per_gpu": n_seq,
                   "G": cfg.G, "B": cfg.B, "M": list(Ms), "output": args.output, "op": args.op,
                   **({"key_quant_scale": args.key_scale, "key_codec_ms": key_ms} if closed else {}),
                   **({"gop_phis": True} if args.gop_phis else {}),
                   "l2": (f"inputs smaller than L2 ({in_mb:.1f} MiB per launch vs {l2_bytes / 2**20:.0f} MiB L2): "
                          f"L2 flushed ({4 * l2_bytes / 2**20:.0f} MiB write) before every launch, outside its "
                          "events; step time = sum of the launches' event times") if small else
                         (f"inputs larger than L2 ({in_mb:.0f} MiB read per launch vs {l2_bytes / 2**20:.0f} MiB L2); no flush"
                          + (f"; the steps rotate over {n_rot} copies of the frames and {n_rot} output buffers "
                             f"({n_rot * in_mb:.0f} MiB of input between two launches on the same copy)" if n_rot > 1 else "")),
                   "parallelism": f"dp{world} (independent sequences per GPU, no collective)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "achieved_event_pairs": achieved_pairs,
                     "time_base": ("event pair around every launch (sum of the launches' mean times)" if (small or closed) else
                                   "the timed region: K steps queued back to back between one event pair; "
                                   "achieved_event_pairs = the same bytes over the attribution pass's per-launch event times (min(K, 20) steps after the region and a 0.5 s pause) "
                                   "(each pair adds the launch latency an event record exposes: ~6.6 us for a K1-shaped launch)"),
                     "traffic": (traffic or {}).get("mean_bytes_per_launch"),
                     "alg_bytes_per_launch": tot_bytes / len(Ms), "traffic_detail": traffic, "peak_source": peak_src,
                     "kernel": "cs_measure_kernel (all launches of the step; alg bytes = frames read once + "
                               + ("fp32 measurements written once)" if gran is None else
                                  "int16 codes + fp32 scales written once; q16frame either stores fp32 y and re-quantises it "
                                  "(8M <= N) or measures twice, reading the frames twice, against this one-read "
                                  "algorithmic count)")},
        "per_M": per_m,
        "gpu_launches": K * (len(Ms) * (3 if args.output == "q16frame" else 1) + (1 if closed else 0)),
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    # oracle leg (rank 0; outside the timed region): parity of the timed outputs, CPU baseline at N=1
    if closed or args.gop_phis:
        line["parity"] = {"ok": None, "how": "not checked here (tests/test_gpu_keys.py covers this variant)"}
    else:
        phis = [synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2) for M in Ms]
        line["parity"] = timed_output_parity(cfg, Ms, phis, frames_h, outs if gran is None else qouts, gran)
    if not args.no_cpu_baseline and world == 1:   # (rank 0 at N=1 only)
        line["cpu_baseline"] = cpu_baseline(cfg, Ms, budget_s=args.cpu_budget, output=args.output)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return line


# ------------------------------------------------------------------------------- f3 adjoint op
def run_adjoint(args, cfg, Ms):
    """--op adjoint: back-projection x0 = Phi^T y of every CS frame of the workload (the measurements
    the encoder produced, resident in HBM), one cs_adjoint launch per M per step."""
    import torch
    import torch.distributed as dist
    import paper_1311_1419_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    n_seq = cfg.S
    frames = torch.from_numpy(synth.gen_video(cfg, streams=range(rank * n_seq, (rank + 1) * n_seq))).to(dev)
    encs, ys, xs = [], [], []
    for M in Ms:
        phi = synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2)
        e = P.Encoder(cfg.W, cfg.H, cfg.G, cfg.B, M, phi)
        y = e.encode_batch(frames)
        encs.append(e)
        ys.append(y)
        xs.append(torch.empty((y.shape[0], cfg.H, cfg.W), dtype=torch.float32, device=dev))
    del frames
    torch.cuda.synchronize(dev)
    if os.environ.get("BENCH_STABLE_INPUTS", "1") != "0":   # the measurements are resident and nothing writes them
        for e in encs:
            e.set_stable_inputs(frames=False, measurements=True)
    torch.cuda.empty_cache()
    stream = torch.cuda.current_stream(dev)

    def launch(i, st=None):
        encs[i].adjoint(ys[i], xs[i], stream if st is None else st)

    ms_total, launch_ms, clk = timed_steps(args, launch, len(Ms), stream, dev, world)
    K = args.steps
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None
    peak, peak_src = load_peaks()
    n_cs = ys[0].shape[0]
    px = n_cs * cfg.W * cfg.H
    per_m, tot_b, tot_ms = {}, 0.0, 0.0
    for i, M in enumerate(Ms):
        avg = statistics.mean(launch_ms[i])
        b = ys[i].numel() * 4 + xs[i].numel() * 4          # y read once + x written once
        per_m[str(M)] = {"ms_median": statistics.median(launch_ms[i]), "ms_mean": avg,
                         "gpix_s": px / (avg * 1e-3) / 1e9, "alg_gbs": b / (avg * 1e-3) / 1e9,
                         "frac_of_peak": b / (avg * 1e-3) / 1e9 / peak, "alg_bytes": b,
                         "tflops_tf32": 2 * 2 * n_cs * encs[i].nblk * M * cfg.B ** 2 / (avg * 1e-3) / 1e12}
        tot_b += b
        tot_ms += avg
    achieved_pairs = tot_b / (tot_ms * 1e-3) / 1e9
    ms_step = ms_total / K
    achieved = tot_b / (ms_step * 1e-3) / 1e9   # time base: the timed region (as the encode op)
    line = {
        "metric": "CS-frame Gpixels/s back-projected (x0 = Phi^T y per block, frame layout)",
        "value": world * len(Ms) * px / (ms_step * 1e-3) / 1e9, "unit": "Gpixel/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 in, tf32 x2 (hi/lo split) -> f32 (tensor core kind::tf32)",
        "data": "synthetic (measurements of the seeded video, synth/)",
        "config": {"workload": args.workload, "op": "adjoint", "W": cfg.W, "H": cfg.H, "T": cfg.T,
                   "streams_per_gpu": n_seq, "B": cfg.B, "M": list(Ms),
                   "l2": "outputs larger than L2 (x is n_cs*H*W*4 bytes per launch); no flush",
                   "parallelism": f"dp{world} (independent sequences per GPU, no collective)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "achieved_event_pairs": achieved_pairs,
                     "time_base": "the timed region (K steps back to back between one event pair); "
                                  "achieved_event_pairs: the attribution pass's per-launch event pairs",
                     "traffic": None, "peak_source": peak_src,
                     "kernel": "cs_adjoint_kernel (alg bytes = fp32 y read once + fp32 x written once)"},
        "per_M": per_m,
        "gpu_launches": K * len(Ms),
        "clocks": clk.summary(),
        "e2e": {"value": None, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "how": "not measured: the adjoint has a device-buffer C-ABI call only"},
    }
    if not args.no_cpu_baseline and world == 1:   # (rank 0 at N=1 only)
        line["cpu_baseline"] = adjoint_cpu_baseline(cfg, Ms, args.cpu_budget)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return line


# ------------------------------------------------------------------------- f2 frame-level op
PAPER_F2 = dict(W=176, H=144, G=5, CR=50, S=64, T=400)   # QCIF, key + 4 CS frames, CS CR 50


def run_frame(args):
    """--op frame: the paper-faithful frame-level measurement y = A vec(F_cs - F_key) (Eq. 1) with
    one dense A (m = round(W*H / 50) = 507), batched over 64 streams x 400 QCIF frames."""
    import torch
    import torch.distributed as dist
    import paper_1311_1419_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    c = PAPER_F2
    W, H, G, S, T = c["W"], c["H"], c["G"], c["S"], c["T"]
    n = W * H
    m = round(n / c["CR"])
    cfg = synth.CONFIGS["C1"].with_(W=W, H=H, G=G, T=T, S=S)
    frames = torch.from_numpy(synth.gen_video(cfg, streams=range(rank * S, (rank + 1) * S))).to(dev)
    A = synth.phi_from_seed(synth.phi_seed(), m, n)
    fe = P.FrameEncoder(W, H, G, m, A)
    y = torch.empty(fe.out_shape(S, T), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def launch(i, st=None):
        fe.encode_batch(frames, y, stream if st is None else st)

    ms_total, launch_ms, clk = timed_steps(args, launch, 1, stream, dev, world)
    K = args.steps
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None
    n_cs = y.shape[0]
    avg = statistics.mean(launch_ms[0])
    flop = 2.0 * m * n * n_cs
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak, peak_src = float(json.load(f)["bf16_tflops"]), "measured bf16 dense burst (MEASURED_PEAKS.json); fp16 rate = bf16 rate"
    except Exception:
        peak, peak_src = 2250.0, "fallback nominal dense fp16 (B200_PROFILING.md)"
    achieved_pairs = flop / (avg * 1e-3) / 1e12
    ms_step = ms_total / K
    achieved = flop / (ms_step * 1e-3) / 1e12   # time base: the timed region (one launch per step)
    px = n_cs * n
    line = {
        "metric": "CS-frame Gpixels/s measured with one frame-level A (Eq. 1, m = n/50)",
        "value": world * px / (ms_step * 1e-3) / 1e9, "unit": "Gpixel/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8 in, fp16 x fp16 -> fp32 (tensor core kind::f16)",
        "data": "synthetic (seeded surveillance-like video, synth/); A seeded N(0,1/m) fp16",
        "config": {"workload": "paper-qcif-cr50", "op": "frame", "W": W, "H": H, "G": G, "m": m, "n": n,
                   "streams_per_gpu": S, "T": T, "cs_frames": n_cs,
                   "l2": f"frames {S * T * n / 2**20:.0f} MiB per launch (> 126 MiB L2); A {m * n * 2 / 2**20:.1f} MiB L2-resident",
                   "parallelism": f"dp{world} (independent sequences per GPU, no collective)"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "achieved_event_pairs": achieved_pairs,
                     "time_base": "the timed region (K steps back to back between one event pair); "
                                  "achieved_event_pairs: the attribution pass's per-launch event pairs",
                     "traffic": None, "peak_source": peak_src,
                     "kernel": "cs_frame_measure_kernel (algorithmic flop = 2 m n per CS frame)"},
        "per_launch_ms": {"mean": avg, "median": statistics.median(launch_ms[0])},
        "gpu_launches": K,
        "clocks": clk.summary(),
        "e2e": {"value": None, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "how": "not measured: the frame-level path has a device-buffer C-ABI call only"},
    }
    # parity of the timed output (outside the timed region): every CS frame of the rank's first stream
    # against the oracle; R24's worst-case bound and the observed max |dy|/S
    import oracle
    y0 = y[: oracle.cs_frame_count(T, G)].double().cpu().numpy()
    yo, So = oracle.measure_frame(frames[0].cpu().numpy(), A, G)
    d = np.abs(y0 - yo)
    rel = np.where(So > 0, d / np.where(So > 0, So, 1.0), 0.0)
    bound = (n / 16 + 16) * 2.0 ** -23
    n_bad = int(((d > bound * So) | ((So == 0) & (y0 != 0))).sum())
    line["parity"] = {"values": int(y0.size), "n_bad": n_bad, "max_rel": float(rel.max()), "bound_rel": bound,
                      "ok": n_bad == 0, "how": "every CS frame of stream 0 of the timed output vs oracle.measure_frame "
                                                "(|dy| <= (n/16+16) 2^-23 S, DESIGN R24)"}
    if not args.no_cpu_baseline and world == 1:   # (rank 0 at N=1 only)
        fr = synth.gen_stream(cfg, 0, T=2 * G)
        t0 = time.perf_counter()
        oracle.measure_frame(fr, A, G, with_scale=False)
        dt = time.perf_counter() - t0
        ncs = oracle.cs_frame_count(2 * G, G)
        line["cpu_baseline"] = {"value": ncs * n / dt / 1e9, "unit": "Gpixel/s", "cores": cpu_threads(),
                                "kind": "oracle", "sample": f"fp64 numpy oracle measure_frame, {ncs} CS frames, {dt:.2f} s"}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return line


def adjoint_cpu_baseline(cfg, Ms, budget_s=15.0):
    """The oracle's adjoint (fp64 numpy) on CS frames of the workload's shape; frames added until
    about half the budget is spent."""
    import oracle
    rng = np.random.default_rng(0)
    nblk = -(-cfg.W // cfg.B) * -(-cfg.H // cfg.B)
    phis = [synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2) for M in Ms]
    n, dt = 0, 0.0
    t0 = time.perf_counter()
    while dt < budget_s / 2 and n < 64:
        for M, phi in zip(Ms, phis):
            oracle.adjoint(rng.normal(size=(1, nblk, M)), phi, cfg.W, cfg.H, cfg.B)
        n += 1
        dt = time.perf_counter() - t0
    px = n * len(Ms) * cfg.W * cfg.H
    return {"value": px / dt / 1e9, "unit": "Gpixel/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"fp64 numpy oracle adjoint, {n} frame(s) of {cfg.W}x{cfg.H} x M in {list(Ms)}, {dt:.2f} s"}


# ------------------------------------------------------------------------------------ oracle arm
def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return os.cpu_count() or 1


def oracle_sample(cfg, Ms, n_gops=1, seed_stream=0, output="f32"):
    """Encode the first n_gops GOPs of one stream with the oracle for every M (and quantise, for
    the f1 outputs); returns (seconds, CS pixels)."""
    import oracle
    T = min(cfg.T, n_gops * cfg.G)
    frames = synth.gen_stream(cfg, seed_stream, T=T)
    phis = [synth.phi_from_seed(synth.phi_seed(), M, cfg.B ** 2) for M in Ms]
    t0 = time.perf_counter()
    nbx = -(-cfg.W // cfg.B)
    for phi in phis:
        y, _ = oracle.encode_stream(frames, phi, cfg.G, cfg.B, with_scale=False)
        if output == "q16frame":
            oracle.quantize_frames(y)
        elif output == "q16row":
            oracle.quantize_frames(y, [(b, min(b + nbx, y.shape[1])) for b in range(0, y.shape[1], nbx)])
    dt = time.perf_counter() - t0
    px = len(Ms) * (T - -(-T // cfg.G)) * cfg.W * cfg.H
    return dt, px


def cpu_baseline(cfg, Ms, budget_s=15.0, output="f32"):
    n_gops, dt, px = 1, 0.0, 0
    while True:
        dt, px = oracle_sample(cfg, Ms, n_gops, output=output)
        if dt * 2 > budget_s or n_gops * cfg.G >= cfg.T:
            break
        n_gops = min(-(-cfg.T // cfg.G), max(n_gops + 1, int(n_gops * budget_s / max(dt, 1e-3) / 2)))
    return {"value": px / dt / 1e9, "unit": "Gpixel/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"fp64 numpy oracle ({'y only' if output == 'f32' else 'y + ' + output}), first {n_gops} GOP(s) = {px // (cfg.W * cfg.H) // len(Ms)} CS "
                      f"frames of one {cfg.W}x{cfg.H} stream x M in {list(Ms)}, {dt:.2f} s"}


def run_reference(args, cfg, Ms):
    rank, world, local = dist_env()
    if rank != 0:
        return None
    if args.warmup > 0:  # one untimed pass (page-in, BLAS thread start-up)
        oracle_sample(cfg, Ms, 1, output=args.output)
    times, pxs = [], []
    for _ in range(args.steps):
        dt, px = oracle_sample(cfg, Ms, 1, output=args.output)
        times.append(dt)
        pxs.append(px)
    ms = 1e3 * sum(times) / len(times)
    value = sum(pxs) / sum(times) / 1e9
    cores = cpu_threads()
    line = {
        "impl": "reference",
        "metric": "CS-frame Gpixels/s encoded (residual vs GOP key + block measurement Y = Phi R)",
        "value": value, "unit": "Gpixel/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded surveillance-like video, synth/)",
        "config": {"workload": args.workload, "W": cfg.W, "H": cfg.H, "T": cfg.T, "G": cfg.G, "B": cfg.B,
                   "M": list(Ms), "output": args.output, "sample_per_step": "first GOP of one stream, every M"},
        "cpu_baseline": {"value": value, "unit": "Gpixel/s", "cores": cores, "kind": "oracle",
                         "sample": "fp64 numpy oracle (y only) on the first GOP of one stream for every M, per step"},
        "e2e": {"value": value, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))
    return line


def self_launch(args, argv):
    """--gpus N > 1 without a torchrun environment: re-run this script under torch.distributed.run with
    N ranks on this node (one process per GPU, rendezvous on 127.0.0.1); rank 0 prints the line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 1) // args.gpus)))
    return subprocess.call(cmd, env=env)


def launcher_check(args):
    """--launcher-check: the multi-rank plumbing without a GPU (gloo): every rank joins, the max over
    ranks of a per-rank 'time' is taken as the timed region does, rank 0 prints n_gpus."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    else:
        ms = 1.0
    if rank == 0:
        print(json.dumps({"launcher_check": True, "n_gpus": world, "max_ms_over_ranks": ms,
                          "streams": [rank * synth.CONFIGS[args.workload].S for rank in range(world)]}))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C4", choices=list(synth.CONFIGS))
    ap.add_argument("--M", default=None, help="comma-separated subset of the config's M values")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-rotate", action="store_true",
                    help="inputs below 2x L2 (C3, C2): flush L2 before every launch instead of rotating copies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-autotune", action="store_true")
    ap.add_argument("--tune-candidates", type=int, default=12)
    ap.add_argument("--op", choices=["encode", "adjoint", "closed_loop", "frame"], default="encode",
                    help="encode (the north-star hot path, default), adjoint (f3 back-projection) or "
                         "closed_loop (f4: key codec + encode against the decoded keys)")
    ap.add_argument("--key-scale", type=float, default=1.0, help="closed_loop: key quantiser scale")
    ap.add_argument("--gop-phis", action="store_true", help="encode: one Phi per GOP index (seed ^ g)")
    ap.add_argument("--output", choices=list(OUTPUTS), default="f32",
                    help="f32 measurements (headline) or 16-bit codes (f1): per-frame or per-row scales")
    ap.add_argument("--tune-file", default=None, help="json of chosen plan indices (read if present, else written)")
    ap.add_argument("--launcher-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:   # not under torchrun: launch the N ranks ourselves
        return self_launch(args, argv)
    if args.launcher_check:
        return launcher_check(args)
    if args.warmup < 3 and args.impl == "ours":
        ap.error("--warmup must be >= 3")
    cfg = synth.CONFIGS[args.workload]
    Ms = tuple(int(m) for m in args.M.split(",")) if args.M else cfg.Ms
    if args.impl == "reference":
        return run_reference(args, cfg, Ms)
    if args.op == "adjoint":
        return run_adjoint(args, cfg, Ms)
    if args.op == "frame":
        return run_frame(args)
    return run_ours(args, cfg, Ms)


if __name__ == "__main__":
    rc = main()
    sys.exit(rc if isinstance(rc, int) else 0)
