#!/usr/bin/env python
"""Benchmark: labelled training pixels/s (fwd + bwd + SGD, whole image) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl mpf|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = one SGD step on a global batch (BASELINE.json configs; R14): every rank runs
mpf_forward_image + mpf_backward_image on its shard of the batch, the flat fp32
gradient is summed over ranks with one NCCL all-reduce (N > 1), then mpf_sgd_step.
Inputs are resident in HBM before the timed region (value); `e2e` repeats the step
through mpf_train_step_host from pinned host buffers (H2D images+labels and the D2H of
the per-image losses inside the timed region).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import mpf_synth as S  # noqa: E402

METRIC = "labelled training pixels/sec (fwd+bwd+SGD, whole-image) at 1/2/4/8 B200"
UNIT = "labelled px/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""
    FIELDS = ("pci.bus_id,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, bus_id: str | None):
        self.bus_id = (bus_id or "").lower()
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def rd():
            for ln in self.proc.stdout:
                self.rows.append([c.strip() for c in ln.split(",")])
        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        if self.bus_id:
            mine = [r for r in rows if self.bus_id.endswith(r[0].lower()[-12:]) or r[0].lower().endswith(self.bus_id[-12:])]
            rows = mine or rows
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _ncu_traffic(workload, kernel, layer):
    """DRAM bytes (read + write) per launch of `kernel` at `layer`, from the committed
    `ncu --set full` capture summary (profiles/ncu_traffic.json, written by
    scripts/ncu_traffic.py from the same kernel at the same config), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            table = json.load(f)
        return table.get(f"{workload}:{kernel}:{layer}")
    except Exception:
        return None


def cpu_baseline(cfg, seconds=12.0, seed=0):
    """The oracle O1 (naive patch-by-patch fp64, as it stands) on a bounded pixel sample
    of one image of the same workload, on this host's cores."""
    import oracle  # test infrastructure: only this leg of bench.py may use it
    threads = oracle.default_threads()
    images, labels = S.make_batch(cfg, [seed])
    params = S.init_params(cfg)
    O = cfg.out_rows * cfg.out_cols
    rng = np.random.default_rng(seed)
    t0 = time.perf_counter()
    pix = rng.choice(O, threads, replace=False).astype(np.int32)
    oracle.o1_image(cfg.layers, cfg.P, params, images[0].astype(np.float64), labels[0], pix=pix,
                    threads=threads, need_probs=False)
    t1 = time.perf_counter() - t0
    reps = max(1, int(seconds / max(t1, 1e-3)))
    n = min(O, threads * reps)
    pix = np.sort(rng.choice(O, n, replace=False)).astype(np.int32)
    t0 = time.perf_counter()
    _, nlab, _, _ = oracle.o1_image(cfg.layers, cfg.P, params, images[0].astype(np.float64), labels[0],
                                    pix=pix, threads=threads, need_probs=False)
    dt = time.perf_counter() - t0
    return {"value": nlab / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"O1 fp64 patch-by-patch fwd+bwd on {n} random output pixels ({nlab} labelled) of one "
                      f"{cfg.H}x{cfg.W} {cfg.name} image, {dt:.1f} s"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle (O1, fp64 patch-by-patch C) timed on the host cores.
    Rank 0 only; other ranks exit without work."""
    if rank != 0:
        return
    import oracle
    threads = oracle.default_threads()
    params = S.init_params(cfg)
    images, labels = S.make_batch(cfg, [0])
    img = images[0].astype(np.float64)
    O = cfg.out_rows * cfg.out_cols
    rng = np.random.default_rng(1)
    per_step = threads * max(1, args.ref_px_per_thread)

    def step(i):
        pix = np.sort(rng.choice(O, per_step, replace=False)).astype(np.int32)
        _, nlab, g, _ = oracle.o1_image(cfg.layers, cfg.P, params, img, labels[0], pix=pix, threads=threads,
                                        need_probs=False)
        return nlab

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    tot = 0
    for i in range(args.steps):
        tot += step(i)
    dt = time.perf_counter() - t0
    v = tot / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"each step: O1 fp64 patch-by-patch fwd+bwd on {per_step} random output "
                                       f"pixels of one {cfg.H}x{cfg.W} {cfg.name} image"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(cfg, world):
    return {"workload": f"{cfg.name}: {cfg.description}; P={cfg.P}, {len(cfg.layers)} layers, "
                        f"{cfg.classes} classes, SGD lr {cfg.lr}",
            "global_batch": cfg.global_batch, "image": [cfg.H, cfg.W], "patch": cfg.P,
            "labelled_px_per_image": cfg.out_rows * cfg.out_cols, "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (per-step working set of tape+deltas >> 126 MB)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4", choices=sorted(S.CONFIGS))
    ap.add_argument("--impl", default="mpf", choices=["mpf", "reference"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the timed steps eagerly")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="multi-rank gradient exchange: pushes into peer memory summed by the SGD kernel "
                         "(default; NCCL if a GPU pair lacks P2P) or bucketed NCCL all-reduces")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-px-per-thread", type=int, default=1)
    ap.add_argument("--profile-json", default="", help="also write the per-kernel table here")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = S.CONFIGS[args.workload]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1302_1690_b200 import dist as D
    from paper_1302_1690_b200.net import MPFNet
    # MPF_BENCH_FUNCTIONAL_1GPU=1: a functional check of the multi-rank code path on a box with
    # one GPU (every rank on cuda:0, gloo instead of NCCL); its numbers are meaningless and it
    # is never used for a reported value
    one_gpu_check = os.environ.get("MPF_BENCH_FUNCTIONAL_1GPU") == "1"
    if one_gpu_check:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun the process group is created at every world size (world 1 included:
    # the NCCL path then runs on one rank, which tests/test_bench_launch.py exercises)
    use_dist = world > 1 or ("LOCAL_RANK" in os.environ and "MASTER_ADDR" in os.environ)
    if use_dist:
        if one_gpu_check:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    B = cfg.global_batch
    if B % world:
        raise SystemExit(f"global batch {B} not divisible by {world} ranks")
    per = B // world
    net = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=per, precision=args.precision, device=dev)
    net.set_params(S.init_params(cfg).astype(np.float32))
    # two global batches of this rank's shard, resident in HBM (inputs cycle between steps)
    pools = []
    for b in range(2):
        idx = D.batch_indices(b, B, world, rank)
        im, lb = S.make_batch(cfg, idx)
        pools.append((torch.tensor(im, device=dev).contiguous(), torch.tensor(lb, device=dev).contiguous(), im, lb))
    counts = []  # labelled pixels of each global batch (all ranks)
    for p in pools:
        c = torch.tensor([float((p[3] != 255).sum())], device=dev, dtype=torch.float64)
        if use_dist:
            dist.all_reduce(c)
        counts.append(float(c.item()))
    stream = torch.cuda.current_stream(dev)
    # the gradient exchange (a7).  Default: peer memory — the library's backward pushes each
    # gradient bucket into every rank's exchange buffer over NVLink as soon as it is final and
    # the SGD kernel sums the ranks' slots (dist.PeerExchange).  Fallback / --exchange nccl: one
    # NCCL all-reduce per bucket started by the gradient-ready hook, waited for before the SGD.
    buckets = None
    peer = None
    exchange_kind = "local"
    if use_dist and not one_gpu_check:
        ok = args.exchange == "peer" and all(
            r == local or torch.cuda.can_device_access_peer(local, r) for r in range(world))
        okt = torch.tensor([1 if ok else 0], device=dev, dtype=torch.int32)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if okt.item():
            try:
                peer = D.PeerExchange(net)
                exchange_kind = "peer"
            except RuntimeError as ex:  # every rank sees the same outcome (PeerExchange agrees)
                print(f"[bench] peer-memory exchange unavailable ({ex}); NCCL all-reduce", file=sys.stderr)
        if peer is None:
            buckets = D.BucketAllReduce(net.grads)
            net.set_grad_hook(buckets)
            exchange_kind = "nccl"
    elif use_dist:
        exchange_kind = "gloo"

    def exchange():
        if peer is not None:
            return  # inside the backward (pushes) and the SGD kernel (sum)
        if buckets is not None:
            buckets.wait()
        else:
            D.allreduce_grads(net.grads)

    def step(i):
        im, lb = pools[i % 2][0], pools[i % 2][1]
        net.train_step(im, lb)  # forward + backward through the C ABI (mpf_train_step)
        exchange()
        net.sgd_step(cfg.lr, 1.0 / B)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    net.check()  # device-side errors (labels, a gradient exchange that timed out) fail the run here
    if use_dist:  # every rank must hold the same parameters after the exchanged SGD steps
        cs = net.params.double().sum().reshape(1)
        lo, hi = cs.clone(), cs.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        if lo.item() != hi.item():
            raise SystemExit(f"ranks disagree on the parameters after warm-up ({lo.item()} vs {hi.item()})")
    # One CUDA graph per input pool (the step's ~170 launches, its side-stream fork/join and
    # the bucketed NCCL all-reduces replayed as one launch); eager launches if capture fails.
    graphs = None
    if not args.no_graph and not one_gpu_check:
        try:
            graphs = []
            for b in range(2):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    step(b)
                graphs.append(g)
            for i in range(2):  # the captured steps run once before timing
                graphs[i].replay()
            torch.cuda.synchronize(dev)
            # keep the graph only where it is faster: it removes per-launch costs (small
            # steps) but its fixed dependency edges can lose some side-stream overlap
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

            def timed(fn):
                c0.record(stream)
                for i in range(4):
                    fn(i)
                c1.record(stream)
                torch.cuda.synchronize(dev)
                return c0.elapsed_time(c1)
            # three alternating rounds of 4 steps each way, best of each (clock drift hits both)
            t_graph, t_eager = float("inf"), float("inf")
            for _ in range(3):
                t_graph = min(t_graph, timed(lambda i: graphs[i % 2].replay()))
                t_eager = min(t_eager, timed(step))
            tg = torch.tensor([t_graph, t_eager], device=dev, dtype=torch.float64)
            if use_dist:
                dist.all_reduce(tg, op=dist.ReduceOp.MAX)
            keep = tg[0].item() <= 0.99 * tg[1].item()
            print(f"[bench] CUDA graph calibration: 4 graph steps {tg[0].item():.3f} ms, 4 eager steps "
                  f"{tg[1].item():.3f} ms -> {'graph' if keep else 'eager'}", file=sys.stderr)
            if not keep:
                graphs = None
        except Exception as ex:  # noqa: BLE001
            print(f"[bench] CUDA graph capture failed ({ex}); eager launches", file=sys.stderr)
            graphs = None
            torch.cuda.synchronize(dev)

    def timed_step(i):
        if graphs is not None:
            graphs[i % 2].replay()
        else:
            step(i)

    bus = None
    try:
        props = torch.cuda.get_device_properties(dev)
        bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
    except Exception:
        pass
    clk = ClockSampler(bus)
    clk.start()
    time.sleep(0.3)
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        timed_step(i)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if use_dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clocks = clk.stop()
    net.check()
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_px = sum(counts[i % 2] for i in range(args.steps))
    value = total_px / (ms_max / 1e3)

    # ---- e2e: the same step through the host-buffer C-ABI call (pinned H2D + loss D2H inside)
    e2e = None
    if not args.no_e2e:
        h_pools = [(torch.tensor(p[2]).pin_memory(), torch.tensor(p[3]).pin_memory()) for p in pools]
        h_loss = torch.zeros(per, dtype=torch.float32).pin_memory()

        def hstep(i):
            hi, hl = h_pools[i % 2]
            net.train_step_host(hi, hl, h_loss, apply_sgd=not use_dist, lr=cfg.lr, grad_scale=1.0 / B)
            if use_dist:
                exchange()
                net.sgd_step(cfg.lr, 1.0 / B)

        for i in range(max(1, args.warmup)):
            hstep(i)
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for i in range(args.steps):
            hstep(i)
        h1.record(stream)
        torch.cuda.synchronize(dev)
        hms = torch.tensor([h0.elapsed_time(h1)], device=dev, dtype=torch.float64)
        if use_dist:
            dist.all_reduce(hms, op=dist.ReduceOp.MAX)
        e2e = {"value": total_px / (float(hms.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h_pools[0][0].numel() * 4 + h_pools[0][1].numel()),
               "d2h_bytes_per_step": int(h_loss.numel() * 4)}

    # ---- roofline of the dominant kernel.  The timed loop overlaps each layer's weight
    # gradient (side stream) with the dgrad / MPF-backward chain, so a kernel's wall time
    # there includes waiting for SMs held by its neighbour.  Per-kernel durations come from
    # the same number of steps run right after it with the weight gradients serialised on
    # the main stream, one CUDA-event pair per launch on its stream.
    from paper_1302_1690_b200 import _lib as L
    net.set_flags(L.MPF_FLAG_SERIAL)
    try:
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        net.profile_begin(200 * max(1, args.steps) + 100)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for i in range(args.steps):
            step(i)
        p1.record(stream)
        torch.cuda.synchronize(dev)
        stats = net.profile_end()
        ser_ms = p0.elapsed_time(p1)
    finally:
        net.set_flags(0)
    peaks, src = _peaks()
    stats.sort(key=lambda r: -r["total_ms"])
    launches = sum(r["launches"] for r in stats)
    dom = stats[0]
    avg_ms = dom["total_ms"] / dom["launches"]
    name = dom["name"]
    tf32_sust = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * 0.5  # TF32 = 1/2 bf16 (nominal ratio)
    if name.endswith("_tc"):
        roof = {"bound": "tensor", "achieved": dom["flops"] / avg_ms / 1e9, "peak": tf32_sust, "unit": "TFLOP/s",
                "peak_source": f"{src} bf16_tflops_sustained x 0.5 (TF32/BF16 nominal ratio)"}
    elif dom["flops"] > 0 and name.startswith(("conv", "dgrad", "wgrad")) and not name.startswith("wgrad_reduce"):
        alu_peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        roof = {"bound": "alu", "achieved": dom["flops"] / avg_ms / 1e9, "peak": alu_peak, "unit": "TFLOP/s",
                "peak_source": "fp32 FFMA: 148 SMs x 128 lanes x 2 flop x sm_max_mhz (DESIGN.md)"}
    else:
        roof = {"bound": "hbm", "achieved": dom["bytes"] / avg_ms / 1e6, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "peak_source": f"{src} hbm_gbs"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = _ncu_traffic(cfg.name, name, dom["layer"])
    roof["kernel"] = f"{name}[layer {dom['layer']}]"
    roof["share_of_step"] = dom["total_ms"] / ser_ms
    roof["measured"] = (f"CUDA events per launch over {args.steps} steps with the weight gradients serialised on "
                        f"the main stream ({ser_ms / args.steps:.2f} ms/step), right after the timed loop")
    roof["algorithmic_per_launch"] = dom["flops"] if roof["bound"] != "hbm" else dom["bytes"]
    # The library counts the positions of the uniform-fragment layout (every fragment padded
    # to the largest one): a few % more than the dense positions the
    # paper's sums run over ((H - rf + 1)(W - rf + 1) per image at that layer).  The stricter
    # fraction counts only those.
    try:
        rr, cc, d = cfg.H, cfg.W, 1
        dense = []
        for Ly in cfg.layers:
            rr, cc = rr - (Ly.k - 1) * d, cc - (Ly.k - 1) * d
            if Ly.kind == S.POOL:
                d *= Ly.k
            dense.append(rr * cc)
        lay = dom["layer"]
        if 0 <= lay < len(dense):
            uni = net.geom.frag[lay + 1] * net.geom.rows[lay + 1] * net.geom.cols[lay + 1]
            roof["dense_positions_per_image"] = dense[lay]
            roof["uniform_fragment_positions_per_image"] = int(uni)
            if roof["bound"] != "hbm" and uni >= dense[lay] > 0:
                roof["frac_dense_positions"] = roof["frac"] * dense[lay] / uni
    except Exception as ex:  # noqa: BLE001 -- a reporting detail must not fail the run
        print(f"[bench] dense-position fraction skipped ({ex})", file=sys.stderr)

    if args.profile_json and rank == 0:
        with open(args.profile_json, "w") as f:
            json.dump({"step_ms": ser_ms / args.steps, "overlapped_step_ms": ms / args.steps, "kernels": stats}, f,
                      indent=1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_seconds)

    if rank == 0:
        any_tc = any(r["name"].endswith("_tc") for r in stats)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "tf32" if any_tc else "f32",
                "data": "synthetic (seeded steel-like images, BASELINE.json shapes)",
                "config": dict(workload_config(cfg, world), cuda_graph=graphs is not None,
                               grad_exchange=exchange_kind), "e2e": e2e,
                "gpu_launches": launches,
                "roofline": roof, "cpu_baseline": cpu, "clocks": clocks}
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
