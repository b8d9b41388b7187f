#!/usr/bin/env python
"""bench.py -- conv2d forward GFLOP/s on B200 (BASELINE.json metric), 1..8 GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--math fp32|tf32] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one pass of the ResNet-50 v1.5 conv stack (53 convs, BASELINE.json configs[4],
DESIGN.md reading R11) over the global batch of 256 images, batch-sharded over the N ranks
(rank r owns images [r*256/N, (r+1)*256/N); no collective on the data path; strong scaling).
Every conv has its own seeded synthetic input and filter (device twin of synth.py) and
runs through conv2d_forward(AUTO): the auto-selector's measured choice per layer.

Rank 0 prints ONE JSON line.  value = total flops of all ranks / max-over-ranks device time.
Timing: W untimed warm-up steps, then K steps each bracketed by CUDA events on the
launching stream, L2 flushed (256 MiB write) before every step outside the events, a
barrier + synchronize on both sides of the timed region; nvidia-smi clocks sampled during
it.  Also reported: roofline of the dominant kernel group, the CPU oracle baseline, the
end-to-end number through the public API with pinned host buffers, launch count.

--impl reference times the CPU oracle (oracle/, the only reference this paper-only run
has) on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1904_04174_b200 import layers as L  # noqa: E402
from paper_1904_04174_b200 import synth  # noqa: E402

METRIC = "conv2d forward GFLOP/s per VGG/ResNet layer, % of B200 peak, 1/2/4/8 GPUs"
GLOBAL_BATCH = 256


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def layer_bytes(l, batch):
    """Algorithmic bytes: touched input + filter + output, fp32."""
    ho = -(-l.rows // l.stride)
    wo = -(-l.cols // l.stride)
    if l.window == 1 and l.stride > 1:
        touched = batch * ho * wo * l.channels  # strided 1x1 reads only the sampled pixels
    else:
        touched = batch * l.rows * l.cols * l.channels
    return 4 * (touched + l.window * l.window * l.channels * l.features + batch * ho * wo * l.features)


def own_flops(l, batch, algo, C):
    """The method's own work for one conv: Winograd F(m x m, 3x3) executes
    2 * alpha^2 * T * C * F multiply-adds-as-flops in its batched GEMM (alpha = m + 2, T = N*ceil(Ho/m)*ceil(Wo/m));
    every other algorithm executes the direct 2*N*Ho*Wo*K^2*C*F."""
    ho = -(-l.rows // l.stride)
    wo = -(-l.cols // l.stride)
    if algo in (C.ALGO_WINOGRAD_F2X2_3X3, C.ALGO_WINOGRAD_F4X4_3X3):
        m = 2 if algo == C.ALGO_WINOGRAD_F2X2_3X3 else 4
        t = batch * (-(-ho // m)) * (-(-wo // m))
        return 2 * (m + 2) ** 2 * t * l.channels * l.features
    return l.flops(batch)


def gemm_kernel_durations(C, convs, ws, flush, tensor_algos, reps=1):
    """Per conv, the mean device duration (ms) of its GEMM-core launch over `reps` replays of the step graph
    with the kernels' %globaltimer stamps on (include/conv2d_debug.h); None for CUDA-core convs.  A launch's
    span = first CTA entry .. last CTA exit, its start clipped to the previous launch's end (PDL overlap)."""
    import torch
    n_gemm = sum(1 for cv in convs if cv["algo"] in tensor_algos)
    if n_gemm == 0:
        return None
    reps = max(1, min(reps, 256 // n_gemm))
    C.conv2d_debug_trace(1)
    try:
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
            cs = torch.cuda.current_stream()
            for _ in range(reps):
                for cv in convs:
                    C.conv2d_forward(cv["p"], C.ALGO_AUTO, cv["x"], cv["w"], cv["y"], ws, ws.numel(), cs)
    finally:
        C.conv2d_debug_trace(0)
    flush.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    t = C.conv2d_debug_trace(-1, read=True)
    rec = 148 * 8
    sums = [0.0] * len(convs)
    k, prev_end = 0, None
    for _ in range(reps):
        for i, cv in enumerate(convs):
            if cv["algo"] not in tensor_algos:
                continue
            r = t[k * rec:(k + 1) * rec]
            k += 1
            ent = [r[j * 8] for j in range(148) if r[j * 8]]
            ext = [r[j * 8 + 7] for j in range(148) if r[j * 8 + 7]]
            if not ent or not ext:
                continue
            start, end = min(ent), max(ext)
            if prev_end is not None and start < prev_end:
                start = prev_end
            sums[i] += (end - start) / 1e6
            prev_end = end
    return [s / reps if cv["algo"] in tensor_algos else None for s, cv in zip(sums, convs)]


def load_traffic(args, math_fp32_or_tf32):
    """ncu DRAM traffic of one timed step at this workload (profiles/<round>_step_traffic*.json, written by
    tools/step_traffic.py from the committed launch list): per GEMM-core launch and for the whole step
    (every launch: transforms, filter prep, reduces included)."""
    out = {"traffic": None}
    if args.math != "fp32":
        return out
    for rnd in ("round2", "round1"):
        tname = f"{rnd}_step_traffic.json" if args.global_batch == 256 else f"{rnd}_step_traffic_b{args.global_batch}.json"
        tpath = os.path.join(ROOT, "profiles", tname)
        if not os.path.exists(tpath):
            continue
        with open(tpath) as fh:
            tj = json.load(fh)
        if not tj.get("gemm_launches") or tj.get("global_batch", 256) != args.global_batch:
            continue
        out["traffic"] = round(tj["gemm_dram_bytes"] / tj["gemm_launches"] / 1e6, 2)
        out["traffic_unit"] = (f"MB per GEMM-core launch, ncu dram__bytes_read.sum+write.sum over one timed step "
                               f"(profiles/{tname}, {tj['gemm_launches']} launches)")
        if "step_dram_bytes" in tj:
            out["traffic_step_gb"] = round(tj["step_dram_bytes"] / 1e9, 3)
            out["traffic_step_note"] = "every launch of the step (transforms, filter prep, reduces included)"
        if "gemm_time_share" in tj:
            out["ncu_gemm_share_of_step"] = round(tj["gemm_time_share"], 4)
        break
    return out


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons, pw = [], [], set(), []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ----------------------------------------------------------------------------- oracle (CPU) legs
def oracle_sample(images: int, math_layers=None):
    """Host inputs for `images` images of every conv of the stack (global images 0..images-1)."""
    import oracle as O
    work = []
    for conv_id, l in L.resnet50_v15_stack():
        x = synth.input_nhwc(images, l.rows, l.cols, l.channels, layer_id=conv_id)
        w = synth.filter_hwcf(l.window, l.window, l.channels, l.features, layer_id=conv_id)
        op = O.Params(images, l.rows, l.cols, l.channels, l.features, l.window, l.window, l.stride, l.stride, O.SAME)
        work.append((op, x, w, l.flops(images)))
    return work


def run_oracle(work, threads):
    import oracle as O
    t0 = time.perf_counter()
    for op, x, w, _ in work:
        O.conv2d(op, x, w, threads=threads)
    return time.perf_counter() - t0


def cpu_baseline(target_s: float = 15.0):
    """The oracle as it stands, on this host's cores, over a bounded sample of the workload."""
    import oracle as O
    O.build()
    threads = os.cpu_count() or 1
    w1 = oracle_sample(1)
    t1 = run_oracle(w1, threads)
    flops1 = sum(f for *_, f in w1)
    images = max(1, min(64, int(target_s / max(t1, 1e-3))))  # 64 images: ~5.6 GB of host tensors
    if images > 1:
        wk = oracle_sample(images)
        t = run_oracle(wk, threads)
        flops = sum(f for *_, f in wk)
    else:
        t, flops = t1, flops1
    return {"value": round(flops / t / 1e9, 3), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
            "sample": f"all 53 convs of the ResNet-50 v1.5 stack on {images} image(s) (global images 0..{images-1}),"
                      f" full oracle incl. double accumulation; {flops/1e9:.2f} GFLOP in {t:.2f} s"}


def config1_leg(args):
    """BASELINE.json configs[0] (N=1, 8x8x4 -> 8x8x8, 3x3, stride 1, SAME): per algorithm the
    GPU time of one conv2d_forward -- the median of single CUDA-graph replays bracketed by events, and the
    per-call time of 1000 back-to-back replays -- next to the oracle's time on this host (cpu_baseline leg:
    1 thread and every core).  Prints one JSON line (not the bench contract line)."""
    import torch
    import oracle as O
    from paper_1904_04174_b200 import conv2d as C
    O.build()
    torch.cuda.set_device(0)
    p0 = C.Params(1, 8, 8, 4, 8, 3, 3, 1, 1, C.PAD_SAME)
    xh = synth.input_nhwc(1, 8, 8, 4, layer_id=1)
    wh = synth.filter_hwcf(3, 3, 4, 8, layer_id=1)
    x, w = torch.from_numpy(xh).cuda(), torch.from_numpy(wh).cuda()
    y = torch.empty(512, device="cuda")
    flops = C.conv2d_flop_count(p0)
    gpu = {}
    for math in (C.MATH_FP32, C.MATH_TF32):
        p = p0.replace(math=math)
        for a in range(1, C.NUM_ALGOS):
            if not C.conv2d_supports(p, a):
                continue
            need = C.conv2d_query_workspace(p, a)
            ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
            for _ in range(5):
                C.conv2d_forward(p, a, x, w, y, ws, ws.numel())
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                C.conv2d_forward(p, a, x, w, y, ws, ws.numel(), torch.cuda.current_stream())
            g1000 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1000, capture_error_mode="thread_local"):
                for _ in range(1000):
                    C.conv2d_forward(p, a, x, w, y, ws, ws.numel(), torch.cuda.current_stream())
            g.replay()
            g1000.replay()
            torch.cuda.synchronize()
            singles = []
            for _ in range(50):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                e1.synchronize()
                singles.append(e0.elapsed_time(e1) * 1e3)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g1000.replay()
            e1.record()
            e1.synchronize()
            per_call = e0.elapsed_time(e1)  # ms for 1000 calls = us per call
            gpu[f"{C.ALGO_NAMES[a]}/{'tf32' if math else 'fp32'}"] = {
                "single_us": round(statistics.median(singles), 2), "back_to_back_us": round(per_call, 3),
                "launches": C.conv2d_launch_count(p, a), "gflops_back_to_back": round(flops / (per_call * 1e3), 2)}
    op = O.Params(1, 8, 8, 4, 8, 3, 3, 1, 1, O.SAME)
    cores = os.cpu_count() or 1
    orc = {}
    for th in (1, cores):
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            O.conv2d(op, xh, wh, threads=th)
            ts.append((time.perf_counter() - t0) * 1e6)
        orc[f"threads_{th}"] = {"median_us": round(statistics.median(ts), 2), "min_us": round(min(ts), 2)}
    print(json.dumps({"config1": {"workload": "BASELINE configs[0]: N=1, 8x8x4, 3x3, F=8, stride 1, SAME",
                                  "flops": flops, "gpu": gpu, "oracle": orc, "cores": cores,
                                  "oracle_note": "oracle/ through ctypes (includes the call overhead), "
                                                 "median of 200 calls"}}), flush=True)
    return 0


def oracle_layers_leg(args):
    """cpu_baseline leg, per layer (the Fig.-1 tables' oracle column): the oracle's GFLOP/s on one image of
    every ResNet-50 set and VGG-16 layer, all host cores; one JSON line."""
    import oracle as O
    O.build()
    cores = os.cpu_count() or 1
    out = {}
    for l in list(L.RESNET50_SETS) + [l for l, _ in L.VGG16_LAYERS]:
        x = synth.input_nhwc(1, l.rows, l.cols, l.channels, layer_id=5000)
        w = synth.filter_hwcf(l.window, l.window, l.channels, l.features, layer_id=5000)
        op = O.Params(1, l.rows, l.cols, l.channels, l.features, l.window, l.window, l.stride, l.stride, O.SAME)
        t0 = time.perf_counter()
        O.conv2d(op, x, w, threads=cores)
        t = time.perf_counter() - t0
        out[l.name] = {"gflops": round(l.flops(1) / t / 1e9, 2), "ms": round(t * 1e3, 2)}
    print(json.dumps({"oracle_layers": out, "cores": cores, "sample": "1 image per layer"}), flush=True)
    return 0


def reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import oracle as O
    O.build()
    threads = os.cpu_count() or 1
    work = oracle_sample(1)
    flops = sum(f for *_, f in work)
    for _ in range(args.warmup):
        run_oracle(work, threads)
    times = [run_oracle(work, threads) for _ in range(args.steps)]
    total = sum(times)
    value = flops * args.steps / total / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64-accumulate",
            "data": "synthetic", "config": workload_config(args, 1),
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
                             "sample": "each step: all 53 convs of the stack on 1 image (global image 0)"},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def self_launch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: re-exec this command under torch.distributed.run with
    N local ranks (one process per GPU; rendezvous on 127.0.0.1) and return its exit status."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def plumbing_arm(args):
    """The multi-rank launch path without a GPU (gloo): the same shard ranges, choice broadcast and
    max-over-ranks timing as the real run; rank 0 prints one JSON line with value null."""
    import torch
    import torch.distributed as dist
    from paper_1904_04174_b200.shard import broadcast_choices, max_over_ranks, shard_range
    rank, world, _ = env_rank()
    if world > 1:
        dist.init_process_group("gloo")
    d = dist if world > 1 else None
    img0, img1 = shard_range(args.global_batch, world, rank)
    names = sorted({l.name for _, l in L.resnet50_v15_stack()})
    chosen = broadcast_choices({nm: (3 + rank, rank) for nm in names}, d, "cpu")
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    x = torch.arange((img1 - img0) * 1000, dtype=torch.float64).sum().item()  # stand-in work, no conv
    t_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, d, "cpu")
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": round(t_ms, 6), "plumbing": True,
                          "config": workload_config(args, img1 - img0),
                          "comm": {"backend": "gloo", "world_size": world},
                          "choices_from_rank0": all(v == (3, 0) for v in chosen.values()), "checksum": x}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def workload_config(args, per_gpu):
    gb = getattr(args, "global_batch", GLOBAL_BATCH)
    return {"workload": "resnet50_v1.5_conv_stack (53 convs, BASELINE configs[4])", "global_batch": gb,
            "per_gpu_batch": per_gpu, "math": "3xtf32 (fp32-faithful)" if args.math == "fp32" else "tf32",
            "algo": ("auto (learned selector, conv2d_predict)" if getattr(args, "predict", False)
                     else "auto (measured: learned top-3 candidates)" if getattr(args, "hybrid", False)
                     else "auto (measured per layer)"), "parallelism": f"batch-shard x{args.gpus}",
            "l2": "flushed before every step (256 MiB write, outside the timed events); step working set ~22 GB",
            "gflop_per_step": round(sum(l.flops(gb) for _, l in L.resnet50_v15_stack()) / 1e9, 3)}


# ----------------------------------------------------------------------------- our arm
def step_trace(args, C, convs, ws, flush):
    """One extra, untimed replay of the step captured with the GEMM-kernel trace on: per launch (= per
    conv), the CTA entry/setup/first-MMA/exit stamps relative to the step's first entry."""
    import torch
    C.conv2d_debug_trace(1)
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
        cs = torch.cuda.current_stream()
        for cv in convs:
            C.conv2d_forward(cv["p"], C.ALGO_AUTO, cv["x"], cv["w"], cv["y"], ws, ws.numel(), cs)
    C.conv2d_debug_trace(0)
    flush.zero_()
    g.replay()
    torch.cuda.synchronize()
    t = C.conv2d_debug_trace(-1, read=True)
    rec = 148 * 8
    out, t0, prev_end, k = [], None, None, 0
    for i, cv in enumerate(convs):
        if cv["algo"] in (C.ALGO_DIRECT, C.ALGO_TILED):  # no GEMM-core launch, no record
            continue
        r = t[k * rec:(k + 1) * rec]
        k += 1
        ctas = [r[j * 8:(j + 1) * 8] for j in range(148) if r[j * 8] != 0]
        if not ctas:
            continue
        start = min(c[0] for c in ctas)
        t0 = start if t0 is None else t0
        end = max(c[7] for c in ctas)
        med = lambda j: statistics.median([c[j] for c in ctas if c[j]]) if any(c[j] for c in ctas) else None
        ent = {"conv": i, "layer": cv["layer"].name, "algo": C.ALGO_NAMES[cv["algo"]], "ctas": len(ctas),
               "start_us": round((start - t0) / 1e3, 2), "span_us": round((end - start) / 1e3, 2),
               "gap_before_us": round((start - prev_end) / 1e3, 2) if prev_end else None}
        for slot, nm in ((1, "setup"), (3, "mma0"), (5, "last_store")):
            m = med(slot)
            ent[nm + "_med_us"] = round((m - start) / 1e3, 2) if m else None
        ent["exit_med_us"] = round((med(7) - start) / 1e3, 2)
        out.append(ent)
        prev_end = end
    with open(args.trace_out, "w") as fh:
        json.dump(out, fh, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--math", choices=["fp32", "tf32"], default="fp32")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of replaying CUDA graphs")
    ap.add_argument("--global-batch", type=int, default=GLOBAL_BATCH,
                    help="analysis only (default = BASELINE config 5's 256)")
    ap.add_argument("--layers-out", default="", help="write the per-layer table (JSON) here")
    ap.add_argument("--save-selection", default="", help="write the tuned selector table here (rank 0)")
    ap.add_argument("--hybrid", action="store_true",
                    help="measure only the learned selector's top 3 candidates per layer (CONV2D_AUTO_HYBRID)")
    ap.add_argument("--predict", action="store_true",
                    help="take the learned selector's choices (conv2d_predict) instead of measuring (analysis)")
    ap.add_argument("--load-selection", default="", help="seed the selector from this table instead of tuning")
    ap.add_argument("--trace-out", default="", help="diagnostics: per-launch GEMM timeline of one extra "
                    "(untimed) graph replay of the step, JSON (include/conv2d_debug.h)")
    ap.add_argument("--verify", action="store_true",
                    help="N>1: gather per-conv output digests of every shard to rank 0 (NCCL) and check them "
                         "bitwise against rank 0 recomputing that shard's images with the same kernels (P11)")
    ap.add_argument("--plumbing", action="store_true",
                    help="CPU-only check of the multi-rank launch path (gloo): shard ranges, choice broadcast, "
                         "max-over-ranks timing; no convolution runs and no value is reported")
    ap.add_argument("--config1", action="store_true",
                    help="BASELINE configs[0]: GPU us per algorithm + the oracle's us (1 thread, all cores)")
    ap.add_argument("--oracle-layers", action="store_true",
                    help="cpu_baseline leg per layer: the oracle's GFLOP/s on one image of every paper layer")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args.gpus)  # one process per GPU, as the driver's torchrun launch does
    if int(os.environ.get("WORLD_SIZE", 1)) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE', 1)} ranks were "
              f"launched", file=sys.stderr)
        return 2
    if args.plumbing:
        return plumbing_arm(args)
    if args.config1:
        return config1_leg(args)
    if args.oracle_layers:
        return oracle_layers_leg(args)
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist
    from paper_1904_04174_b200 import conv2d as C

    rank, world, local = env_rank()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_1904_04174_b200.shard import broadcast_choices, max_over_ranks, shard_range
    img0, img1 = shard_range(args.global_batch, world, rank)
    B = img1 - img0
    math = C.MATH_FP32 if args.math == "fp32" else C.MATH_TF32
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- resident inputs (device generator, global image offsets -> shards are exact slices)
    stack = L.resnet50_v15_stack()
    convs = []
    ws_bytes = 0
    for conv_id, l in stack:
        p = C.Params(**l.params(B), math=math)
        (n, ho, wo, f), _ = C.conv2d_output_shape(p)
        per_img = l.rows * l.cols * l.channels
        x = torch.empty(B * per_img, dtype=torch.float32, device=dev)
        C.conv2d_synth_fill(x, x.numel(), synth.stream_key(synth.SEED, conv_id, synth.ROLE_INPUT),
                            img0 * per_img, 0)
        w = torch.empty(l.window * l.window * l.channels * l.features, dtype=torch.float32, device=dev)
        C.conv2d_synth_fill(w, w.numel(), synth.stream_key(synth.SEED, conv_id, synth.ROLE_FILTER), 0, 0)
        y = torch.empty(n * ho * wo * f, dtype=torch.float32, device=dev)
        ws_bytes = max(ws_bytes, C.conv2d_query_workspace(p, C.ALGO_AUTO))
        convs.append(dict(id=conv_id, layer=l, p=p, x=x, w=w, y=y, flops=C.conv2d_flop_count(p),
                          bytes=layer_bytes(l, B)))
    ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    # ---- auto-selection (measured, once per distinct layer); rank 0's choices (algorithm + tuned
    #      variant) broadcast so every rank runs the same kernels (off the timed path)
    chosen = {}
    tune0 = time.perf_counter()
    if args.hybrid:  # time only the learned selector's top candidates per layer (CONV2D_AUTO_HYBRID)
        C.conv2d_set_auto_policy(C.AUTO_HYBRID)
    C.conv2d_set_autotune_flush(flush)  # cache-cold candidate timings, as in the timed step
    if args.load_selection:
        C.conv2d_load_selection(args.load_selection)
    for cv in convs:
        key = cv["layer"].name
        if key not in chosen:
            sel = C.conv2d_selected(cv["p"]) if args.load_selection else None
            if sel is None and args.predict:  # the learned selector's choice, no measurement (conv2d_predict)
                sel, v = C.conv2d_predict(cv["p"])
                C.conv2d_set_selected(cv["p"], sel)
                if sel in (C.ALGO_IMPLICIT_GEMM, C.ALGO_MATMUL_1X1):
                    C.conv2d_set_variant(cv["p"], sel, v)
            chosen[key] = sel if sel is not None else C.conv2d_autotune(cv["p"], cv["x"], cv["w"], cv["y"], ws,
                                                                        ws.numel())
    if args.save_selection and rank == 0:
        C.conv2d_save_selection(args.save_selection)
    C.conv2d_set_autotune_flush(None)
    C.conv2d_set_auto_policy(C.AUTO_MEASURE)
    tune_s = time.perf_counter() - tune0
    gemm_like = (C.ALGO_IMPLICIT_GEMM, C.ALGO_MATMUL_1X1)
    chosen = {k: (a, C.conv2d_get_variant(next(cv["p"] for cv in convs if cv["layer"].name == k), a)
                  if a in gemm_like else 0) for k, a in chosen.items()}
    chosen = broadcast_choices(chosen, dist if world > 1 else None, dev)  # (algorithm, variant) pairs
    for cv in convs:
        a, v = chosen[cv["layer"].name]
        C.conv2d_set_selected(cv["p"], a)
        if a in gemm_like:
            C.conv2d_set_variant(cv["p"], a, v)
        cv["algo"] = a
        cv["launches"] = C.conv2d_launch_count(cv["p"], C.ALGO_AUTO)

    def step(evs=None):
        for i, cv in enumerate(convs):
            if evs is not None:
                evs[i][0].record(stream)
            C.conv2d_forward(cv["p"], C.ALGO_AUTO, cv["x"], cv["w"], cv["y"], ws, ws.numel(), stream)
            if evs is not None:
                evs[i][1].record(stream)

    for _ in range(max(args.warmup, 1)):
        flush.zero_()
        step()
    torch.cuda.synchronize()

    # ---- timed region
    # CUDA graphs: one captured graph per timed step (the 53 conv2d_forward calls), replayed on the
    # launching stream.  The timed graphs carry NO per-conv events: an event node between two kernels
    # costs ~9 us at the boundary (measured: 2.39 vs 1.90 ms/step at b32), so per-conv times come from
    # separate instrumented replays right after the timed region (same graphs + events per conv).
    ev_step = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ev_conv = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in convs]
               for _ in range(args.steps)]
    graphs, graphs_ev = None, None
    if not args.no_graph:
        try:
            cap = torch.cuda.Stream()
            graphs, graphs_ev = [], []
            for k in range(args.steps):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                    cs = torch.cuda.current_stream()
                    for cv in convs:
                        C.conv2d_forward(cv["p"], C.ALGO_AUTO, cv["x"], cv["w"], cv["y"], ws, ws.numel(), cs)
                graphs.append(g)
                ev_conv[k] = [(torch.cuda.Event(enable_timing=True, external=True),
                               torch.cuda.Event(enable_timing=True, external=True)) for _ in convs]
                ge = torch.cuda.CUDAGraph()
                with torch.cuda.graph(ge, stream=cap, capture_error_mode="thread_local"):
                    cs = torch.cuda.current_stream()
                    for i, cv in enumerate(convs):
                        ev_conv[k][i][0].record(cs)
                        C.conv2d_forward(cv["p"], C.ALGO_AUTO, cv["x"], cv["w"], cv["y"], ws, ws.numel(), cs)
                        ev_conv[k][i][1].record(cs)
                graphs_ev.append(ge)
            for g in graphs + graphs_ev:  # warm replays
                g.replay()
            torch.cuda.synchronize()
            ev_conv[0][0][0].elapsed_time(ev_conv[0][0][1])  # timing of external events works?
        except Exception as exc:  # fall back to eager launches (reported in config)
            print(f"[bench] CUDA graph capture unavailable ({exc!r}); timing eager launches", file=sys.stderr)
            graphs, graphs_ev = None, None
            ev_conv = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                        for _ in convs] for _ in range(args.steps)]

    def timed_region():
        clocks = ClockSampler(local)
        barrier()
        torch.cuda.synchronize()
        if rank == 0:
            clocks.start()
            time.sleep(0.3)
        torch.cuda.nvtx.range_push("bench_timed")  # ncu --nvtx --nvtx-include "bench_timed/" selects these
        wall0 = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()
            ev_step[k][0].record(stream)
            if graphs is not None:
                graphs[k].replay()
            else:
                step()
            ev_step[k][1].record(stream)
        torch.cuda.synchronize()
        wall_s = time.perf_counter() - wall0
        torch.cuda.nvtx.range_pop()
        barrier()
        return wall_s, (clocks.stop() if rank == 0 else None)

    wall, clk = timed_region()
    # a run that saw hardware / thermal slowdown is re-measured once (rank 0 decides for every rank)
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    redo = int(rank == 0 and clk is not None and bool(bad & set(clk.get("reasons") or [])))
    if world > 1:
        flag = torch.tensor([redo], dtype=torch.int32, device=dev)
        dist.broadcast(flag, 0)
        redo = int(flag.item())
    if redo:
        first = clk
        wall, clk = timed_region()
        if clk is not None:
            clk["remeasured_after"] = first.get("reasons")
    t_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev_step), dist if world > 1 else None, dev)
    flops_step_all = sum(cv["flops"] for cv in convs) * world
    value = flops_step_all * args.steps / (t_ms / 1e3) / 1e9

    # ---- per-conv times: K instrumented replays (events around every conv), L2 flushed before each
    for k in range(args.steps):
        flush.zero_()
        if graphs_ev is not None:
            graphs_ev[k].replay()
        else:
            step(ev_conv[k])
    torch.cuda.synchronize()
    per_conv_ms = [statistics.mean(ev_conv[k][i][0].elapsed_time(ev_conv[k][i][1]) for k in range(args.steps))
                   for i in range(len(convs))]
    peaks, peak_src = load_peaks()
    tf32_peak = peaks["bf16_tflops"] / 2.0             # nominal TF32 : BF16 = 1 : 2 (B200_PROFILING.md)
    useful_peak = tf32_peak / 3.0 if math == C.MATH_FP32 else tf32_peak  # 3 MMAs per product in 3xTF32
    hbm = peaks["hbm_gbs"]
    # Own-work accounting: a Winograd conv is credited with the multiplies it
    # executes, 2*alpha^2*T*C*F for its batched tensor-core GEMM, not the direct-convolution flops the
    # metric `value` uses (reading R8).  Every other conv's own work is its direct flops.
    for cv in convs:
        cv["own_flops"] = own_flops(cv["layer"], B, cv["algo"], C)
    tensor_algos = (C.ALGO_IMPLICIT_GEMM, C.ALGO_MATMUL_1X1, C.ALGO_WINOGRAD_F2X2_3X3, C.ALGO_WINOGRAD_F4X4_3X3)
    # dominant kernel = the tcgen05 GEMM core (gemm2sm_kernel / halo_kernel): one launch per conv whose
    # algorithm is implicit_gemm / matmul_1x1 / winograd.  Its per-launch device durations come from the
    # kernels' own %globaltimer stamps (include/conv2d_debug.h) in instrumented replays of the same step
    # graph right after the timed region (L2 flushed before each); the step time is the CUDA-event time.
    kd = gemm_kernel_durations(C, convs, ws, flush, tensor_algos, reps=min(args.steps, 4)) if rank == 0 else None
    step_ms = t_ms / args.steps
    grp = [cv for cv in convs if cv["algo"] in tensor_algos]
    roof = {"bound": "tensor", "unit": "TFLOP/s", "peak": round(useful_peak, 1)}
    if kd and grp:
        k_ms = sum(kd[i] for i, cv in enumerate(convs) if cv["algo"] in tensor_algos)
        k_flops = sum(cv["own_flops"] for cv in grp)
        ach = k_flops / (k_ms / 1e3) / 1e12
        roof.update({"achieved": round(ach, 2), "frac": round(ach / useful_peak, 4),
                     "kernel": f"GEMM core (persistent 2-CTA tcgen05 gemm2sm_kernel / halo_kernel), {len(grp)} launches "
                               f"per step ({len(grp)} of {len(convs)} convs), {100 * k_ms / step_ms:.1f}% of the step",
                     "kernel_ms_per_step": round(k_ms, 3), "kernel_share_of_step": round(k_ms / step_ms, 4),
                     "timing": "per-launch device durations (first CTA entry to last CTA exit, %globaltimer) of the "
                               "GEMM-core launches in min(K,4) instrumented replays of the step graph after the timed "
                               "region, L2 flushed; step time = CUDA events on the launching stream"})
    else:
        k_flops = sum(cv["own_flops"] for cv in convs)
        ach = k_flops / (step_ms / 1e3) / 1e12
        roof.update({"achieved": round(ach, 2), "frac": round(ach / useful_peak, 4),
                     "kernel": "whole step (no GEMM-core launch timeline available on this rank)"})
    roof["flop_accounting"] = ("own work: batched-GEMM multiplies 2*alpha^2*T*C*F for Winograd convs "
                               "(alpha^2 = 16 / 36; transforms not counted as flops), direct flops 2*N*Ho*Wo*K^2*C*F "
                               "for the rest; `value` stays direct-normalised (reading R8)")
    roof["peak_source"] = (f"{peak_src} bf16 burst {peaks['bf16_tflops']} TF/s /2 (TF32)"
                           + (" /3 (3xTF32 useful flops)" if math == C.MATH_FP32 else ""))
    traffic = load_traffic(args, math)
    roof.update(traffic)
    # whole-step roofline: sum over convs of max(own flops / peak, algorithmic bytes / HBM)
    roof_ms = sum(max(cv["own_flops"] / (useful_peak * 1e12), cv["bytes"] / (hbm * 1e9)) * 1e3 for cv in convs)
    roof["step_roofline_ms"] = round(roof_ms, 3)
    roof["step_frac"] = round(roof_ms / step_ms, 4)
    roof["step_achieved_own_tflops"] = round(sum(cv["own_flops"] for cv in convs) / (step_ms / 1e3) / 1e12, 2)
    roof["algorithmic_gb_per_step"] = round(sum(cv["bytes"] for cv in convs) / 1e9, 3)

    layers_table = []
    seen = {}
    for cv, ms in zip(convs, per_conv_ms):
        nm = cv["layer"].name
        if nm in seen:
            seen[nm]["ms"].append(ms)
            continue
        seen[nm] = {"layer": nm, "tuple": [cv["layer"].window, cv["layer"].stride, cv["layer"].rows,
                                           cv["layer"].cols, cv["layer"].channels, cv["layer"].features],
                    "batch": B, "algo": C.ALGO_NAMES[cv["algo"]], "ms": [ms], "flops": cv["flops"],
                    "own_flops": cv["own_flops"], "bytes": cv["bytes"]}
        layers_table.append(seen[nm])
    for r in layers_table:
        t = statistics.mean(r["ms"])
        r["us"] = round(1e3 * t, 2)
        r["gflops"] = round(r["flops"] / (t / 1e3) / 1e9, 1)
        r["own_tflops"] = round(r["own_flops"] / (t / 1e3) / 1e12, 2)
        r["gbs"] = round(r["bytes"] / (t / 1e3) / 1e9, 1)
        rl = max(r["own_flops"] / (useful_peak * 1e12), r["bytes"] / (hbm * 1e9)) * 1e3
        r["roofline_frac"] = round(rl / t, 3)
        r["bound"] = "tensor" if r["own_flops"] / (useful_peak * 1e12) >= r["bytes"] / (hbm * 1e9) else "hbm"
        r["count"] = len(r["ms"])
        del r["ms"]

    launches = sum(cv["launches"] for cv in convs) * args.steps

    if args.trace_out and rank == 0:
        step_trace(args, C, convs, ws, flush)

    # ---- end to end through the public API: pinned host -> device, forward, device -> host
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, C, convs, ws, stream, world, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()

    verify = None
    if args.verify:
        verify = verify_shards(args, C, convs, ws, stream, world, rank, dev)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(t_ms / args.steps, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32" if math == C.MATH_FP32 else "tf32",
                "data": "synthetic (seeded splitmix64 uniform[-1,1), device-generated)",
                "config": dict(workload_config(args, B), cuda_graph=graphs is not None,
                               selection_s=round(tune_s, 2)),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk, "wall_s_timed": round(wall, 3),
                "pct_of_peak": round(100 * roof["step_achieved_own_tflops"] / useful_peak, 2),
                "comm": {"backend": dist.get_backend() if world > 1 else None, "world_size": world}}
        if verify is not None:
            line["verify"] = verify
        if args.layers_out:
            with open(args.layers_out, "w") as f:
                json.dump({"bench": line, "layers": layers_table}, f, indent=1)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def output_digests(convs):
    """Per conv: two exact integer digests of the output's bit patterns (plain and position-weighted
    int64 sums; integer addition is associative, so the digest itself is deterministic)."""
    import torch
    rows = []
    for cv in convs:
        bits = cv["y"].view(torch.int32).long()
        wgt = torch.arange(bits.numel(), device=bits.device, dtype=torch.int64) % 1021 + 1
        rows.append(torch.stack([bits.sum(), (bits * wgt).sum()]))
    return torch.stack(rows)


def verify_shards(args, C, convs, ws, stream, world, rank, dev):
    """P11 across ranks (--verify, off the timed path): every rank's output digests are all-gathered to
    rank 0 (NCCL), which regenerates each other rank's images from their global indices, runs the same
    kernels (rank 0's broadcast choices; same per-GPU batch, so the same launch plan) and requires
    bit-identical digests."""
    import torch
    import torch.distributed as dist
    from paper_1904_04174_b200.shard import shard_range
    mine = output_digests(convs)
    if world == 1:
        return {"ranks_checked": 0, "note": "single rank: nothing to cross-check"}
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    ok, checked = True, 0
    if rank == 0:
        for r in range(1, world):
            img0, _ = shard_range(args.global_batch, world, r)
            for cv in convs:
                l = cv["layer"]
                per_img = l.rows * l.cols * l.channels
                C.conv2d_synth_fill(cv["x"], cv["x"].numel(), synth.stream_key(synth.SEED, cv["id"], synth.ROLE_INPUT),
                                    img0 * per_img, 0)
            for cv in convs:
                C.conv2d_forward(cv["p"], C.ALGO_AUTO, cv["x"], cv["w"], cv["y"], ws, ws.numel(), stream)
            torch.cuda.synchronize()
            ok = ok and bool(torch.equal(output_digests(convs), parts[r]))
            checked += 1
    flag = torch.tensor([int(ok)], dtype=torch.int32, device=dev)
    dist.broadcast(flag, 0)
    return {"ranks_checked": checked, "bitwise": bool(flag.item()), "digest": "int64 sums of output bits per conv",
            "how": "NCCL all_gather of shard digests; rank 0 recomputes each shard's images with the same kernels"}


def run_e2e(args, C, convs, ws, stream, world, dev):
    """Same metric through the public API with host buffers: every step copies each conv's input
    from pinned host memory, runs conv2d_forward, and reads each output back to pinned host memory.
    Copies and compute are pipelined over three streams (H2D, compute, D2H)."""
    import torch
    import torch.distributed as dist
    # per distinct layer one pinned host input/output (the step still moves every conv's bytes)
    host_in, host_out = {}, {}
    for cv in convs:
        nm = cv["layer"].name
        if nm not in host_in:
            host_in[nm] = torch.empty(cv["x"].numel(), dtype=torch.float32, pin_memory=True)
            host_in[nm].copy_(cv["x"])
            host_out[nm] = torch.empty(cv["y"].numel(), dtype=torch.float32, pin_memory=True)
    s_h2d = torch.cuda.Stream()
    s_d2h = torch.cuda.Stream()
    h2d_bytes = sum(cv["x"].numel() * 4 for cv in convs)
    d2h_bytes = sum(cv["y"].numel() * 4 for cv in convs)
    # device staging: two input slots per size class would save memory; the resident buffers are reused
    ev_in = [torch.cuda.Event() for _ in convs]
    ev_done = [torch.cuda.Event() for _ in convs]

    def e2e_step():
        for i, cv in enumerate(convs):
            with torch.cuda.stream(s_h2d):
                if i > 0:
                    s_h2d.wait_event(ev_done[i - 1])  # keep at most one conv of copies ahead
                cv["x"].copy_(host_in[cv["layer"].name], non_blocking=True)
                ev_in[i].record(s_h2d)
            stream.wait_event(ev_in[i])
            C.conv2d_forward(cv["p"], C.ALGO_AUTO, cv["x"], cv["w"], cv["y"], ws, ws.numel(), stream)
            ev_done[i].record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_done[i])
                host_out[cv["layer"].name].copy_(cv["y"], non_blocking=True)
        stream.wait_stream(s_d2h)

    e2e_step()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    from paper_1904_04174_b200.shard import max_over_ranks
    t = max_over_ranks(e0.elapsed_time(e1), dist if world > 1 else None, dev)
    flops = sum(cv["flops"] for cv in convs) * world * steps
    return {"value": round(flops / (t / 1e3) / 1e9, 1), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d_bytes,
            "d2h_bytes_per_step": d2h_bytes, "steps": steps, "ms_per_step": round(t / steps, 3),
            "path": "pinned host -> cudaMemcpyAsync -> conv2d_forward(AUTO) -> cudaMemcpyAsync -> pinned host, "
                    "3 streams pipelined"}


if __name__ == "__main__":
    sys.exit(main())
