#!/usr/bin/env python
"""Benchmark: CaffeNet training images/sec on B200 (BASELINE.json metric).

One step = one synthetic mini-batch through the whole hot path: device batch
gather -> forward (lowering + tcgen05 GEMM per conv/FC layer, fused
bias/ReLU, pooling, softmax-CE) -> backward (weight/data-gradient GEMMs,
col2im, pooling, bias gradients) -> [NCCL allreduce of the gradient when
N > 1] -> fused momentum-SGD update.  Weak scaling: every GPU processes
--batch images per step.

    python bench.py                                  # N = 1, CaffeNet b=256, TF32
    torchrun --nproc-per-node N bench.py --gpus N    # one rank per GPU
    python bench.py --impl reference                 # the reference CPU path (oracle port)
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

# stdout carries exactly one JSON line: keep the real stdout for it and send
# everything else that writes to fd 1 (NCCL's version banner, library chatter) to stderr.
os.environ["NCCL_DEBUG"] = os.environ.get("BENCH_NCCL_DEBUG", "WARN")
# Measured on 4x B200 (profiles/README.md): the per-layer gradient allreduces,
# overlapped with the backward, run 6% faster over ring/tree than over NVLS.
os.environ.setdefault("NCCL_NVLS_ENABLE", "0")
_JSON_FD = os.dup(1)
os.dup2(2, 1)


def emit(obj) -> None:
    os.write(_JSON_FD, (json.dumps(obj) + "\n").encode())

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CaffeNet train images/sec at 1/2/4/8 B200 per g; conv GEMM % tensor peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--net", default="caffenet")
    ap.add_argument("--batch", type=int, default=256, help="images per GPU per step")
    ap.add_argument("--precision", default="tf32", choices=["tf32", "3xtf32"])
    ap.add_argument("--n-examples", type=int, default=1024)
    ap.add_argument("--cpu-batch", type=int, default=0,
                    help="images per --impl reference step (rounded to whole images per core; "
                         "default 4 per core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--eta", type=float, default=0.01)
    ap.add_argument("--mu", type=float, default=0.9)
    ap.add_argument("--lam", type=float, default=5e-4)
    ap.add_argument("--profile-out", default="", help="write per-GEMM timing breakdown (json)")
    ap.add_argument("--groups-nccl", dest="groups_p2p", action="store_false",
                    help="--groups: NCCL all-to-all rounds instead of the default per-layer exchanges "
                         "over NVLink peer memory (copy-engine DMA)")
    ap.add_argument("--groups-overlap", action="store_true",
                    help="--groups: layer-aligned shards, gradient exchange overlapped with the backward")
    ap.add_argument("--nccl-allreduce", dest="p2p", action="store_false",
                    help="N > 1: NCCL allreduce + separate update instead of the default fused "
                         "gradient reduce + update over peer memory (comm.PeerUpdate)")
    ap.add_argument("--merged-fc", action="store_true",
                    help="N > 1: FC layers on rank 0 for the global batch (PAPER.md:936-959)")
    ap.add_argument("--groups", type=int, default=1,
                    help="compute groups g (g > 1: groups.GroupRuntime, deterministic round-robin "
                         "async schedule; momentum retuned per g by Theorem 1)")
    return ap.parse_args()


# ------------------------------------------------------------------ util --
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            # nvidia-smi takes a moment to start: wait for its first sample so the
            # (short) timed region is inside the sampled window
            t0 = time.time()
            while time.time() - t0 < 3.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].isdigit():
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("", "[N/A]"))}


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def tf32_peak(peaks: dict) -> tuple[float, str]:
    """Dense TF32 tensor peak: half the measured dense bf16 rate (the B200
    datasheet ratio 1.1 / 2.25 PF).  The BURST figure: bench.py times every
    conv GEMM launch on its own (CUDA events around each launch, clocks at
    1965 MHz, ~300 W), not inside a power-capped back-to-back loop -- the
    measurement the sustained figure describes (its clocks fell to 1290 MHz)."""
    if "bf16_tflops" in peaks:
        return peaks["bf16_tflops"] / 2.0, "MEASURED_PEAKS bf16_tflops (burst) / 2 (tf32 = 1/2 bf16 dense)"
    return 1590.0 / 2.0, "fallback 1.59 PF/s bf16 (B200_PROFILING.md) / 2"


def tf32_peak_sustained(peaks: dict):
    if "bf16_tflops_sustained" in peaks:
        return peaks["bf16_tflops_sustained"] / 2.0
    return None


def measure_tf32_peak(dev) -> dict:
    """cuBLAS TF32 GEMM, 8192^3 (torch.matmul with TF32 enabled), best of 10
    launches timed alone with CUDA events -- the measured TF32 counterpart of
    MEASURED_PEAKS' cuBLAS bf16 burst figure (same method, same box, same run)."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        g = torch.Generator(device=dev).manual_seed(0)
        a = torch.randn(n, n, device=dev, generator=g)
        b = torch.randn(n, n, device=dev, generator=g)
        for _ in range(3):
            torch.matmul(a, b)
        best = float("inf")
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return {"tflops": 2.0 * n ** 3 / (best * 1e-3) / 1e12, "ms": best,
                "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS TF32), best of 10, CUDA events"}
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:   # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_operands(net, b: int, seed: int) -> list:
    """Every GEMM layer of ``net`` at batch b as the reference would see it:
    (kind, input, weights, stride, pad) with synthetic float64 operands of the
    layer's shape (conv: NCHW input + OIHW kernel; fc: (b, f) + (f, out))."""
    rng = np.random.default_rng(seed)
    out = []
    for g in net.geometry():
        L = g.layer
        if L.kind == "conv":
            c, n, _ = g.in_shape
            out.append(("conv", rng.standard_normal((b, c, n, n)),
                        0.01 * rng.standard_normal((L.d_out, c, L.k, L.k)), L.stride, L.pad,
                        g.index == 0))
        elif L.kind == "fc":
            f = int(np.prod(g.in_shape))
            out.append(("fc", rng.standard_normal((b, f)), 0.01 * rng.standard_normal((f, L.d_out)),
                        1, 0, False))
    return out


def reference_step_seconds(ops, cores: int) -> tuple[float, float, list]:
    """Time the reference's own operators on this host:
    conv_lowered(D, K, spec, b_p=b, workers=cores) per conv layer
    (tensors.py:222-256, 128-block float64 einsum GEMMs) and flat @ W per FC
    layer (problems.py:218).  The reference has no backward for these layers,
    so the step is extrapolated the paper's way: backward =
    weight gradient + data gradient = 2 x forward GEMM, 1 x for the first
    layer (no data gradient).  Returns (forward s, extrapolated step s, per-layer s)."""
    from oracle import refcnn as R

    fwd = step = 0.0
    per = []
    for kind, D, Wk, s, p, first in ops:
        t0 = time.perf_counter()
        if kind == "conv":
            R.conv_lowered(D, Wk, s, p, b_p=D.shape[0], workers=cores)
        else:
            _ = D @ Wk
        t = time.perf_counter() - t0
        fwd += t
        step += t * (2.0 if first else 3.0)
        per.append(t)
    return fwd, step, per


def cpu_baseline(net, batch: int, seed: int) -> dict:
    """The reference algorithm (oracle port of tensors.py / problems.py,
    float64 NumPy) on all of this host's cores at the benchmark's own batch."""
    cores = host_cores()
    ops = reference_operands(net, batch, seed)
    fwd, step, per = reference_step_seconds(ops, cores)
    return {"value": batch / step, "unit": "images/s", "cores": cores, "kind": "port",
            "sample": f"one {net.name} step at b={batch} (the full per-GPU batch): the reference's "
                      f"conv_lowered(b_p={batch}, workers={cores}) per conv layer + flat @ W per FC layer, "
                      f"timed ({fwd:.1f} s forward); backward extrapolated as 2x forward "
                      f"(1x for conv1: weight gradient only), PAPER.md:1822 accounting",
            "seconds": step, "forward_seconds": fwd,
            "layer_forward_seconds": [round(t, 4) for t in per], "cpu_model": cpu_model()}


# ------------------------------------------------------------ reference --
def run_reference(args):
    from paper_1606_04487_b200 import nets

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    net = nets.get(args.net)
    cores = host_cores()
    # Each step is a bounded sample of the workload: the same per-layer
    # reference operators as cpu_baseline at bsz images, 4 whole images per
    # worker thread by default (with a single image per thread the einsum
    # partitions run ~2x slower per image on this code path; from 4 up the
    # per-image cost is flat, so the sample agrees with the full b=256 pass).
    mult = max(1, args.cpu_batch // cores) if args.cpu_batch else 4
    bsz = cores * mult
    steps = max(1, args.steps)
    ops = reference_operands(net, bsz, args.seed)
    for _ in range(max(0, args.warmup)):
        reference_step_seconds(ops, cores)
    tot = fwd_tot = 0.0
    for _ in range(steps):
        fwd, st, per = reference_step_seconds(ops, cores)
        tot += st
        fwd_tot += fwd
    value = steps * bsz / tot
    sample = (f"each step: {args.net} at b={bsz} ({mult} image(s) per core; a bounded sample of the "
              f"b={args.batch}-per-GPU workload): the reference's conv_lowered(b_p={bsz}, "
              f"workers={cores}) per conv layer + flat @ W per FC layer, float64, timed "
              f"({fwd_tot / steps:.2f} s forward per step); backward extrapolated as 2x forward "
              f"(1x for conv1), PAPER.md:1822 accounting")
    cb = {"value": value, "unit": "images/s", "cores": cores, "kind": "port", "sample": sample,
          "seconds": tot, "cpu_model": cpu_model()}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * tot / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(args, args.gpus, net),   # the same workload as our arm
            "sample": sample, "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)


def arm_config(args, world, net) -> dict:
    """The workload both arms report (bench contract: same config, metric, unit)."""
    b, s, c = args.batch, net.in_size, net.in_channels
    return {"workload": f"{args.net} train step, b={b} per GPU, synthetic {s}x{s}x{c}, g=1",
            "net": args.net, "per_gpu_batch": b, "global_batch": b * world, "g": 1,
            "parallelism": f"dp{world}" + ("+merged-fc" if getattr(args, "merged_fc", False) and world > 1
                                           else "+p2p" if getattr(args, "p2p", False) and world > 1
                                           else "+nccl" if world > 1 else ""),
            "precision": args.precision, "l2": l2_note(net, b)}


def l2_note(net, b) -> str:
    """Whether one step's working set exceeds the 126 MB L2; if it does not,
    run_ours flushes L2 (256 MB write) between timed steps."""
    acts = sum(int(np.prod(g.out_shape)) for g in net.geometry())
    est = 4 * b * acts * 2 + 20 * net.dim          # activations + grads, W/V/G/w_read traffic
    if est > 126e6:
        return f"working set ~{est / 1e9:.1f} GB per step > 126 MB L2 (no flush needed)"
    return (f"working set ~{est / 1e6:.0f} MB per step fits in L2: L2 flushed (256 MB write) "
            "between timed steps, each step timed with its own events")


# ------------------------------------------------------------------ ours --
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1606_04487_b200 import _abi, nets
    from paper_1606_04487_b200.problems import CNNProblem, DeviceBatch, HostBatch
    from paper_1606_04487_b200.sgd import Hyperparams, SGDState

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    net = nets.get(args.net)
    b = args.batch
    _abi.load()

    if args.groups > 1:
        return run_groups(args, net, dev, world, rank, local)

    # Public API: CNNProblem (synthetic dataset resident in HBM, distinct per
    # rank) + DeviceSession (W, V in HBM; data parallel over NCCL when N > 1).
    s, c = net.in_size, net.in_channels
    prob = CNNProblem(net, n_examples=args.n_examples, seed=args.seed * 1000 + rank,
                      labels="uniform", precision=args.precision, device=dev)
    hp = Hyperparams(eta=args.eta, mu=args.mu, lam=args.lam, b=b)
    sess = prob.device_session(SGDState.fresh(np.zeros(1)), hp,
                               process_group=dist.group.WORLD if world > 1 else None,
                               merged_fc=args.merged_fc and world > 1,
                               p2p=args.p2p and world > 1 and not args.merged_fc)
    gw = torch.Generator(device=dev)
    gw.manual_seed(args.seed)                     # identical initial model on every rank
    sess.W = 0.01 * torch.randn(net.dim, generator=gw, device=dev)
    sess.V = torch.zeros_like(sess.W)
    eng = sess.engine
    total = args.warmup + args.steps
    rng = np.random.default_rng(np.random.SeedSequence(args.seed, spawn_key=(1, rank)))
    idx_all = torch.from_numpy(rng.integers(0, args.n_examples, size=(total, b))).to(dev)

    def step(i):
        sess.step(DeviceBatch(idx_all[i]))

    # libomni launches per step, counted by the library on the first (eager)
    # warm-up step; later steps replay the same launches from a CUDA graph
    n0 = _abi.query("omni_launch_count")
    step(0)
    launches_per_step = _abi.query("omni_launch_count") - n0
    for i in range(1, args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    st = torch.cuda.current_stream()
    flush = "fits in L2" in l2_note(net, b)
    if not flush:   # one step's working set exceeds L2: time the K steps back to back
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(args.warmup, total):
            step(i)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    else:           # small nets: flush L2 between steps (outside the per-step events)
        scrub = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > L2
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for j, i in enumerate(range(args.warmup, total)):
            scrub.zero_()
            evs[j][0].record(st)
            step(i)
            evs[j][1].record(st)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(z) for a, z in evs)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = args.steps * b * world / (ms / 1000.0)
    loss_now = sess.last_loss()

    # ---- per-GEMM breakdown (one instrumented step, after the timed region):
    # CUDA events around every conv / FC GEMM launch (explicit or implicit).
    # Serial chains here so every launch is timed alone (no stream overlap).
    eng.timer, eng.overlap = [], False
    torch.cuda.synchronize()
    reps = 3
    for r in range(reps):
        step(total - 1)
    torch.cuda.synchronize()
    records, eng.timer, eng.overlap = eng.timer, None, True
    per_step = len(records) // reps
    conv_ms = fc_ms = 0.0
    rows = []
    for M, N, Kd, kind, a0, a1 in records:
        t = a0.elapsed_time(a1)
        if kind == "conv":
            conv_ms += t / reps
        else:
            fc_ms += t / reps
        rows.append({"M": M, "N": N, "K": Kd, "kind": kind, "ms": t,
                     "tflops": 2.0 * M * N * Kd / (t * 1e9)})
    conv_flops_step = net.conv_flops_per_image() * b
    achieved = conv_flops_step / (conv_ms * 1e-3) / 1e12 if conv_ms > 0 else 0.0
    peaks = measured_peaks()
    bf16_half, bf16_src = tf32_peak(peaks)
    tf32_meas = measure_tf32_peak(dev)
    # roofline denominator: the TF32 GEMM peak measured here (cuBLAS, burst);
    # 3xTF32 issues three tf32 MMAs per product, so its peak is a third of that
    peak = tf32_meas["tflops"] / (3.0 if args.precision == "3xtf32" else 1.0)
    peak_src = ("cuBLAS TF32 8192^3 measured in this run (burst), "
                + ("/ 3 (3xTF32: three tf32 MMAs per product)" if args.precision == "3xtf32" else "of measured"))
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "r02_traffic_summary.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            ts = json.load(f)
        if ts.get("net") == args.net and ts.get("per_gpu_batch") == b and ts.get("precision") == args.precision:
            traffic = ts["conv_gemm_dram_bytes_per_step"]
            traffic_src = ("DRAM bytes (read+write) of the conv GEMM launches of one step, " + ts["source"])
    if args.profile_out and rank == 0:
        with open(args.profile_out, "w") as f:
            json.dump({"gemms_one_step": rows[:per_step], "conv_gemm_ms": conv_ms,
                       "fc_gemm_ms": fc_ms, "step_ms": ms / args.steps}, f, indent=1)

    # ---- e2e: the same public call with HOST buffers (pinned H2D in the timed region)
    e2e = None
    if not args.no_e2e:
        # two pinned host batches, alternated: every step copies a full batch in
        gh = torch.Generator().manual_seed(rank)
        host = [HostBatch(torch.randn((b, s, s, c), generator=gh).pin_memory(),
                          torch.randint(0, net.classes, (b,), generator=gh,
                                        dtype=torch.int32).pin_memory()) for _ in range(2)]
        # K steps like the device-timed loop: the first step's copy has nothing to
        # overlap with (pipeline fill) and is amortised over the same window
        n_e2e = max(5, args.steps)
        for rep in range(2):   # warm-up pass, then the timed pass
            if rep == 1:
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
            sess.prefetch(host[0])
            fut = None
            for i in range(n_e2e if rep else 3):
                hb = host[i % 2]
                sess.step(hb)                     # consumes the prefetched copy
                sess.prefetch(host[(i + 1) % 2])  # next batch's H2D overlaps this step
                nxt = sess.loss_future()          # D2H of this step's loss, async
                if fut is not None:
                    _ = fut.result()              # previous step's loss on the host
                fut = nxt
            sess.step(host[(n_e2e if rep else 3) % 2])   # drain the last prefetch
            _ = fut.result()
            _ = sess.last_loss()
        torch.cuda.synchronize()
        n_e2e += 1
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": n_e2e * b * world / dt, "unit": "images/s",
               "h2d_bytes_per_step": host[0].X.numel() * 4 + host[0].y.numel() * 4,
               "d2h_bytes_per_step": 4,
               "path": "CNNProblem.device_session(): prefetch(HostBatch(pinned X, y)) on a copy "
                       "stream overlapping step(); every step's loss read on the host via "
                       "loss_future() (async D2H, read one step later)"}

    # the reference's own call shapes through the drop-in API (float64 NCHW
    # host batches; reported beside e2e, not the headline): run_sync
    # (sgd.py:210-256, device session, full-dataset loss sampled every 5 steps)
    # and the TrainingProblem.grad + sgd_step pair a user's loop calls
    dropin = None
    if rank == 0 and world == 1 and not args.no_e2e:
        dropin = measure_dropin(net, b, args, prob, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(net, b, args.seed)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
            "config": arm_config(args, world, net),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic (Gaussian images, uniform labels, random-init weights)",
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes per step",
                         "peak_cublas_tf32_measured": tf32_meas,
                         "peak_bf16_half": bf16_half, "frac_of_bf16_half": achieved / bf16_half,
                         "bf16_half_source": bf16_src,
                         "peak_nominal_tf32_dense": 1100.0, "frac_of_nominal": achieved / 1100.0,
                         "peak_sustained_tf32": tf32_peak_sustained(peaks),
                         "frac_of_sustained": (achieved / tf32_peak_sustained(peaks)
                                               if tf32_peak_sustained(peaks) else None),
                         "traffic_source": traffic_src,
                         "algorithmic": f"{net.conv_flops_per_image() / 1e9:.4f} GFLOP/img conv FW+BW x {b} img",
                         "kernel": "conv GEMMs (gemm_tf32_kernel: implicit im2col + explicit layer 1)",
                         "peak_source": peak_src, "conv_gemm_ms_per_step": conv_ms,
                         "fc_gemm_ms_per_step": fc_ms,
                         "conv_gemm_share_of_step": conv_ms / (ms / args.steps)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "dropin_api": dropin,
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_source": "omni_launch_count() delta over one eager step x steps "
                                   "(graph replays launch the same kernels)",
            "clocks": clk,
            "loss_after": loss_now,
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def measure_dropin(net, b, args, prob, dev) -> dict:
    """images/s through the reference-shaped API: (1) run_sync for 10 steps
    (device session; full-dataset loss every 5 steps, the reference's
    sampling option), (2) problem.grad(W, (X, y)) with X a float64 NCHW host
    array + sgd_step on float64 host state -- the per-call host<->device
    traffic of the drop-in boundary included."""
    import torch

    from paper_1606_04487_b200.sgd import Hyperparams, SGDState, StopRule, run_sync, sgd_step

    hp = Hyperparams(eta=args.eta, mu=args.mu, lam=args.lam, b=b)
    state = SGDState.fresh(0.01 * np.random.default_rng(args.seed).standard_normal(net.dim))
    torch.cuda.synchronize()
    run_sync(prob, hp, state, StopRule(max_steps=2), seed=args.seed, sample_interval=2)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run_sync(prob, hp, state, StopRule(max_steps=10), seed=args.seed, sample_interval=5)
    torch.cuda.synchronize()
    rs = 10 * b / (time.perf_counter() - t0)
    rng = np.random.default_rng(args.seed)
    X = rng.standard_normal((b, net.in_channels, net.in_size, net.in_size))
    y = rng.integers(0, net.classes, size=b)
    st = state
    g = prob.grad(st.W, (X, y))                     # warm-up
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        g = prob.grad(st.W, (X, y))
        st = sgd_step(st, hp, g, st.W)
    ga = reps * b / (time.perf_counter() - t0)
    return {"run_sync_images_per_s": rs, "grad_sgd_step_images_per_s": ga,
            "path": "run_sync(CNNProblem, ...) 10 steps (device session, full loss every 5); "
                    "problem.grad(W_f64, (X_f64 NCHW, y)) + sgd_step(float64 state) on host arrays"}


def run_groups(args, net, dev, world, rank, local):
    """g compute groups of k = N/g GPUs (groups.GroupRuntime): one round = g
    master updates; every GPU processes --batch images per round."""
    import torch
    import torch.distributed as dist

    from paper_1606_04487_b200.cluster import ExecutionPlan, momentum_for_groups
    from paper_1606_04487_b200.groups import CudaBackend, GroupRuntime
    from paper_1606_04487_b200.problems import CNNProblem
    from paper_1606_04487_b200.sgd import Hyperparams

    if not dist.is_initialized():
        raise SystemExit("--groups > 1 needs torchrun with N divisible by g")
    plan = ExecutionPlan(world, args.groups)
    mu = momentum_for_groups(plan.g, args.mu)
    hp = Hyperparams(eta=args.eta, mu=mu, lam=args.lam, b=args.batch * plan.k)
    prob = CNNProblem(net, n_examples=args.n_examples, seed=args.seed, precision=args.precision,
                      device=dev)
    gw = torch.Generator(device=dev)
    gw.manual_seed(args.seed)
    W0 = 0.01 * torch.randn(net.dim, generator=gw, device=dev)
    rt = GroupRuntime(plan, CudaBackend(prob, args.batch), hp, W0, args.n_examples, args.seed,
                      overlap=args.groups_overlap, p2p=args.groups_p2p)
    rt.run(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    rt.run(args.steps)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    t = torch.tensor([ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = args.steps * args.batch * world / (ms / 1000.0)
    if rank == 0:
        st_ = [e.staleness for e in rt.events[plan.g:]]
        emit({
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic (Gaussian images, uniform labels, random-init weights)",
            "config": {"workload": f"{args.net} train, g={plan.g} compute groups of k={plan.k} GPUs, "
                                   f"b={args.batch} per GPU (group batch {hp.b}), deterministic "
                                   f"round-robin async schedule", "net": args.net,
                       "per_gpu_batch": args.batch, "global_batch": args.batch * world, "g": plan.g,
                       "k": plan.k, "mu": mu, "parallelism": f"{plan.g} groups x dp{plan.k}"
                       + ("+p2p" if args.groups_p2p else "+nccl"),
                       "step": "one round = g master updates"},
            "staleness_mean": float(np.mean(st_)) if st_ else 0.0,
            "gpu_launches": None, "clocks": clk, "e2e": None, "cpu_baseline": None,
            "roofline": None})
    rt.close()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
