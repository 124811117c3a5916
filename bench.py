#!/usr/bin/env python
"""Benchmark of the FTK alignment hot path (arXiv:1905.12317) on B200.

Metric (BASELINE.json): inner products / s = N_im * N_tm * N_t * n_gamma / time, on config c5
("8-GPU scale": n=256, 8192 images x 4096 templates, 797 shifts, 512 rotations), templates sharded
over N GPUs with an all-gather of per-image bests (strong scaling: the job is fixed).

One step = one pass of the whole hot path over the batch:
ring-FFT load of images and templates from polar samples resident in HBM, Steps 1-3 with the fused
max/argmax epilogue, and (N > 1) the NCCL all-gather + merge of per-image bests.  The plan (S0) is
built before timing.  `e2e` repeats the step through the C ABI from pinned HOST buffers with
the host->device copies and the device->host read of the bests inside the timed region.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ftk|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ftk", choices=["ftk", "reference"])
    ap.add_argument("--engine", default="tc", choices=["tc", "simt"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--images", type=int, default=0, help="override N_im (debug only; the metric uses the config)")
    ap.add_argument("--templates", type=int, default=0)
    ap.add_argument("--n-gamma", type=int, default=0,
                    help="rotations per (pair, shift); 0 = n_psi (the configs). > n_psi: zero-padded Step 2 (NEXT-3)")
    ap.add_argument("--pixels", action="store_true",
                    help="inputs are n x n pixel images; each step runs the NUFFT front end (Eq. Ahattrap, NEXT-2) "
                         "before Steps 1-3 (no e2e / cpu_baseline legs)")
    ap.add_argument("--marginal-tau", type=float, default=0.0,
                    help="> 0: time the marginalization epilogue (log sum exp(X / tau) per pair, NEXT-3) instead "
                         "of max / argmax (1 GPU; not the headline metric)")
    ap.add_argument("--eps", type=float, default=0.0, help="override the config's eps (debug only)")
    ap.add_argument("--workspace-gb", type=float, default=0.0, help="fixed pair-block workspace (debug only)")
    ap.add_argument("--ctf-defoci", default="",
                    help="comma-separated defoci [Angstrom]: CTF-parameterized kernel (NEXT-4, reading R24); "
                         "the metric counts every (pair, shift, rotation, defocus) (no e2e / cpu_baseline legs)")
    return ap.parse_args()


METRIC = "inner products/s (pairs x shifts x rotations)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.limit")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._p = None
        self._t = None

    def start(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self._p = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._p.kill()
        if self._t is not None:
            self._t.join(timeout=2)
        return self.summary()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[4 + k].lower() == "active"})
        def num(k):
            v = []
            for r in self.rows:
                try:
                    v.append(float(r[k]))
                except (ValueError, IndexError):
                    pass
            return v
        pw, pl = num(2), num(8)
        capped = sum(1 for r in self.rows if r[7].lower() == "active")
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w": statistics.median(pw) if pw else None, "power_limit_w": max(pl) if pl else None,
                "power_cap_frac": capped / len(self.rows)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return None


def host_description():
    """nproc, CPU model and the BLAS thread count the oracle runs with."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import threadpoolctl
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")}
                for d in threadpoolctl.threadpool_info()]
    except Exception:  # noqa: BLE001
        blas = None
    return {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
            else None, "cpu_model": model, "blas": blas}


def cpu_baseline(cfg, imgs_cpu, tpls_cpu, k_nodes, seconds_budget=15.0):
    """The float64 oracle (as it stands) on a bounded sample of the same workload, on this host's cores."""
    from oracle import fb, ftk, kernel_svd as ks
    plan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi,
                         n_nodes=96)
    a = fb.fb_coeffs(imgs_cpu)
    b = fb.fb_coeffs(tpls_cpu)
    n_t, n_psi = plan.shifts.shape[0], cfg.n_psi
    done_pairs = 0
    t0 = time.perf_counter()
    ni, nj = a.shape[0], b.shape[0]
    chunk_i, chunk_j = 2, 8
    for i0 in range(0, ni, chunk_i):
        for j0 in range(0, nj, chunk_j):
            ftk.ftk_best(a[i0:i0 + chunk_i], b[j0:j0 + chunk_j], plan, chunk_i=chunk_i, chunk_j=chunk_j)
            done_pairs += min(chunk_i, ni - i0) * min(chunk_j, nj - j0)
            if time.perf_counter() - t0 > seconds_budget:
                break
        if time.perf_counter() - t0 > seconds_budget:
            break
    dt = time.perf_counter() - t0
    ips = done_pairs * n_t * n_psi / dt
    try:
        import threadpoolctl
        thr = max((d.get("num_threads", 1) for d in threadpoolctl.threadpool_info()), default=1)
    except Exception:  # noqa: BLE001
        thr = os.cpu_count()
    # the brute-force definition (oracle/brute.py, Eq. Xdg discretized: no Bessel / SVD / FFT) at sampled
    # (pair, shift, rotation) points, time-bounded (the brute-force rate beside the FTK rate)
    from oracle import brute, quadrature
    kq, wq = quadrature.radial_rule(cfg.n_k, cfg.k_max)
    shifts = synth.shift_list(cfg)
    rng = np.random.default_rng(1)
    nbf, tb0 = 0, time.perf_counter()
    while time.perf_counter() - tb0 < 3.0:
        i, j = int(rng.integers(0, ni)), int(rng.integers(0, nj))
        tt, rr = rng.integers(0, n_t, 50), rng.integers(0, n_psi, 50)
        brute.brute_points(imgs_cpu[i], tpls_cpu[j], kq, wq, shifts, tt, rr)
        nbf += 50
    dtb = time.perf_counter() - tb0
    return {"value": ips, "unit": "inner products/s", "cores": int(thr), "kind": "oracle",
            "sample": f"{cfg.name}: {done_pairs} (image, template) pairs x {n_t} shifts x {n_psi} rotations, "
                      f"float64 numpy oracle (FB coeffs + plan excluded), {dt:.1f} s",
            "brute_force": {"value": nbf / dtb, "unit": "inner products/s",
                            "sample": f"{nbf} random (pair, shift, rotation) points of the same sample, "
                                      f"oracle/brute.py (8 n_k n_psi flop per inner product), {dtb:.1f} s"},
            "host": host_description()}


def run_reference(args):
    """--impl reference: the CPU oracle is this tier's reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.config(args.config)
    from oracle import fb, ftk, kernel_svd as ks, quadrature
    k, _ = quadrature.radial_rule(cfg.n_k, cfg.k_max)
    plan = ks.build_plan(cfg.n, cfg.K, synth.delta_max(cfg), synth.shift_list(cfg), cfg.eps, cfg.n_k, cfg.n_psi,
                         n_nodes=96)
    ni, nj = {"tiny": (4, 4), "c2": (4, 16), "c3": (2, 16), "c4": (1, 4), "c5": (2, 8)}[cfg.name]
    imgs, _ = synth.draw_items(cfg, "images", range(ni), k)
    tpls, _ = synth.draw_items(cfg, "templates", range(nj), k)
    n_t = plan.shifts.shape[0]
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        a, b = fb.fb_coeffs(imgs), fb.fb_coeffs(tpls)
        ftk.ftk_best(a, b, plan, chunk_i=2, chunk_j=8)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    per_step = ni * nj * n_t * cfg.n_psi
    value = per_step * len(times) / sum(times)
    try:
        import threadpoolctl
        thr = max((d.get("num_threads", 1) for d in threadpoolctl.threadpool_info()), default=1)
    except Exception:  # noqa: BLE001
        thr = os.cpu_count()
    sample = f"{cfg.name}: {ni}x{nj} pairs x {n_t} shifts x {cfg.n_psi} rotations per step (float64 oracle)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "inner products/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "n_k": cfg.n_k, "n_psi": cfg.n_psi, "N_t": n_t,
                       "eps": cfg.eps, "pairs_per_step": ni * nj},
            "cpu_baseline": {"value": value, "unit": "inner products/s", "cores": int(thr), "kind": "oracle",
                             "sample": sample, "host": host_description()},
            "e2e": {"value": value, "unit": "inner products/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_1905_12317_b200 as pkg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # the library's own NCCL communicator: ftk_align all-gathers + merges the per-image bests itself
        # (torch.distributed only carries the 128-byte unique id)
        comm = pkg.NcclComm.from_group(local)
    dev = f"cuda:{local}"
    cfg = synth.config(args.config, **({"eps": args.eps} if args.eps > 0 else {}))
    ni = args.images or cfg.N_im
    nj = args.templates or cfg.N_tm
    shifts = synth.shift_list(cfg)
    n_t = shifts.shape[0]
    engine = pkg.ENGINE_TC if args.engine == "tc" else pkg.ENGINE_SIMT
    defoci = [float(x) for x in args.ctf_defoci.split(",") if x.strip()]
    filters = None
    if defoci:
        filters = synth.ctf_filters(pkg.radial_rule(cfg.n, cfg.K, cfg.n_k, 0)[0], defoci)
        n_t *= len(defoci)                      # virtual shifts (tau, t)
        args.no_e2e = args.no_cpu_baseline = True
    plan = pkg.FTKPlan(cfg.n, cfg.K, synth.delta_max(cfg), shifts, cfg.eps, n_k=cfg.n_k, n_psi=cfg.n_psi,
                       device=local, rank=rank, world=world, engine=engine, n_gamma=args.n_gamma, filters=filters,
                       workspace_bytes=int(args.workspace_gb * (1 << 30)), nccl_comm=comm)
    n_gamma = plan.info["n_gamma"]
    k, w = plan.radial()
    # synthetic inputs generated on the device (seeded), resident in HBM
    if args.pixels:
        imgs, _ = synth.draw_pixel_items(cfg, "images", range(ni), backend="torch", device=dev)
        tpls, _ = synth.draw_pixel_items(cfg, "templates", range(nj), backend="torch", device=dev)
        args.no_e2e = args.no_cpu_baseline = True
    else:
        imgs, _ = synth.draw_items(cfg, "images", range(ni), k, backend="torch", device=dev)
        tpls, _ = synth.draw_items(cfg, "templates", range(nj), k, backend="torch", device=dev)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def step():
        if args.pixels:
            plan.load_images_pixels(imgs, stream=stream)
            plan.load_templates_pixels(tpls, stream=stream)
        else:
            plan.load_images(imgs, stream=stream)
            plan.load_templates(tpls, stream=stream)
        if args.marginal_tau > 0:
            return plan.align_marginal(args.marginal_tau, stream=stream)
        if world > 1:
            return pkg.distributed_align(plan, stream=stream)
        return plan.align(stream=stream)["best"]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    plan.set_profiling(True)
    sampler = ClockSampler(local)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kt_acc = {}
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        best = step()
        # per-kernel device times of this step (events recorded by the library on its stream)
        for kname, (ms, cnt) in plan.kernel_times().items():
            a = kt_acc.setdefault(kname, [0.0, 0])
            a[0] += ms
            a[1] += cnt
        plan.set_profiling(True)  # reset event pool for the next step
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    plan.set_profiling(False)
    dt_ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([dt_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt_ms = float(t.item())
    total_ips = float(ni) * nj * n_t * n_gamma
    value = total_ips * args.steps / (dt_ms / 1e3)

    # ---- roofline of each hot-path kernel; the dominant one (largest device time in the timed region)
    #      is the line's "roofline"
    info = plan.info
    pairs_local = ni * info["n_templates_local"]
    peaks = measured_peaks()
    try:  # DRAM bytes per pair of each kernel from the committed ncu captures (same config only)
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        tj = {}

    def roof(kern):
        k_ms, k_cnt = kt_acc.get(kern, [0.0, 0])
        avg_s = k_ms / max(k_cnt, 1) / 1e3
        per_launch = pairs_local * args.steps / max(k_cnt, 1)     # pairs one launch processes
        traffic = None
        if tj.get("config") == cfg.name and kern in tj.get("bytes_per_pair", {}):
            traffic = tj["bytes_per_pair"][kern] * per_launch
        r = {"kernel": kern, "launches": k_cnt, "avg_launch_ms": avg_s * 1e3, "traffic": traffic,
             "traffic_unit": "bytes/launch"}
        if kern == "step2":
            # HBM-bound on STAGING bytes: the method's own HBM traffic is ~0 per inner product (SURVEY 8(d):
            # inputs only); Step 2 reads the staged Zhat' (n_psi x H_plus complex fp32) and writes the staged
            # Step-3 operand (n_gamma x K3 real columns, fp16 hi + lo) -- an implementation cost, counted here
            byts = (8.0 * cfg.n_psi * info["H_plus"] + 4.0 * n_gamma * info["K3"]) * per_launch
            peak = peaks["hbm_gbs"] if peaks else 7000.0
            achieved = byts / avg_s / 1e9 if avg_s > 0 else None
            r.update({"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                      "bytes_per_launch": byts, "bytes_kind": "staging (not algorithmic: SURVEY 8(d))",
                      "peak_source": "measured HBM copy GB/s (MEASURED_PEAKS.json)" if peaks
                      else "fallback 7000 GB/s (B200_PROFILING.md)",
                      "note": "staging bytes per pair 8 n_psi H_plus (read Zhat') + 4 n_gamma K3 (write fp16 hi/lo)"})
        else:
            if kern == "step3":
                flops = 2.0 * n_t * n_gamma * info["K3"] * per_launch           # real GEMM, K = 2 H_plus - H0
            else:
                flops = 8.0 * cfg.n_psi * info["H_plus"] * cfg.n_k * per_launch  # complex GEMM over k_m
            achieved = flops / avg_s / 1e12 if avg_s > 0 else None
            if engine == pkg.ENGINE_TC:
                bound, peak_src = "tensor", "measured bf16 sustained (MEASURED_PEAKS.json) x 1 (fp16 dense = bf16 dense, B200_PROFILING.md)"
                peak = peaks["bf16_tflops_sustained"] if peaks else 1400.0
                if not peaks:
                    peak_src = "fallback 1.4 PF/s sustained (B200_PROFILING.md)"
            else:
                bound = "alu"
                mhz = (peaks or {}).get("sm_max_mhz", 1965.0)
                peak = 148 * 128 * 2 * mhz * 1e6 / 1e12   # fp32 FMA lanes x 2 flop x clock
                peak_src = "derived: 148 SM x 128 FP32 lanes x 2 x sm_max_mhz"
            r.update({"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "flops_per_launch": flops,
                      "peak_source": peak_src})
            if engine == pkg.ENGINE_TC and kern == "step3":
                rows = 128 * info["s3_rtiles"]
                issued = 3.0 * 2.0 * rows * info["s3_cols"] * info["K3p"] * per_launch
                r["tensor_issued_tflops"] = issued / avg_s / 1e12 if avg_s > 0 else None
                r["traffic_algorithmic"] = 4.0 * 128 * info["s3_rtiles"] * info["K3p"] * per_launch
                r["note"] = ("achieved = algorithmic flops 2*N_t*n_gamma*K3 per pair (minimal real Step-3 GEMM) / launch "
                             "time; tensor_issued_tflops counts the MMAs actually issued (fp16x3 = 3 products, +-delta "
                             "symmetry halves the rows, tile padding)")
            elif kern == "step1":
                if engine == pkg.ENGINE_TC:
                    s1_rows = ((info["H_plus"] + 1) // 2 * 2) * 2   # generated rows per template (Re/Im per slot)
                    issued = 3.0 * 2.0 * s1_rows * 2 * cfg.n_k * cfg.n_psi * per_launch
                    r["tensor_issued_tflops"] = issued / avg_s / 1e12 if avg_s > 0 else None
                r["note"] = ("achieved = algorithmic flops 8 n_psi H_plus n_k per pair (complex Step-1 GEMM) / launch time; "
                             "tensor_issued_tflops counts the fp16x3 MMAs issued (3 products, Re/Im rows of the padded slots)")
        r["frac"] = (r["achieved"] / r["peak"]) if r.get("achieved") else None
        return r

    kerns = [k2 for k2 in ("step1", "step2", "step3") if kt_acc.get(k2, [0, 0])[1] > 0]
    dom = max(kerns, key=lambda c: kt_acc[c][0]) if kerns else "step3"
    roofline = roof(dom)
    roofline["all_kernels"] = {k2: {f: roof(k2).get(f) for f in ("bound", "achieved", "peak", "unit", "frac",
                                                                   "avg_launch_ms", "tensor_issued_tflops")
                                    if roof(k2).get(f) is not None} for k2 in kerns}
    launches = sum(v[1] for v in kt_acc.values())
    # whole-step tensor floor: the step's tensor work at the measured sustained bf16 (= fp16) peak, in the minimal
    # (algorithmic) and in the issued (fp16x3, padded tiles) form, against the measured step time
    if engine == pkg.ENGINE_TC:
        pairs_step = float(pairs_local)
        alg = pairs_step * (8.0 * cfg.n_psi * info["H_plus"] * cfg.n_k + 2.0 * n_t * n_gamma * info["K3"])
        s1_rows = ((info["H_plus"] + 1) // 2 * 2) * 2      # generated Step-1 rows per template (Re/Im per slot)
        issued = pairs_step * 3.0 * (2.0 * s1_rows * 2 * cfg.n_k * cfg.n_psi +
                                     2.0 * 128 * info["s3_rtiles"] * info["s3_cols"] * info["K3p"])
        pk = (peaks["bf16_tflops_sustained"] if peaks else 1400.0) * 1e12
        step_s = dt_ms / args.steps / 1e3
        roofline["step_tensor_floor"] = {
            "algorithmic_tflop_per_step": alg / 1e12, "issued_tflop_per_step": issued / 1e12,
            "floor_ms_algorithmic": 1e3 * alg / pk, "floor_ms_issued": 1e3 * issued / pk,
            "frac_algorithmic": (alg / pk) / step_s, "frac_issued": (issued / pk) / step_s,
            "peak_source": "measured bf16 sustained (MEASURED_PEAKS.json) = fp16 dense rate" if peaks else "fallback 1.4 PF/s"}

    # ---- end to end through the C ABI from pinned host buffers
    e2e = None
    if not args.no_e2e:
        imgs_h = torch.empty(imgs.shape, dtype=imgs.dtype, pin_memory=True)
        tpls_h = torch.empty(tpls.shape, dtype=tpls.dtype, pin_memory=True)
        imgs_h.copy_(imgs)
        tpls_h.copy_(tpls)
        lo, hi = rank * nj // world, (rank + 1) * nj // world
        del imgs, tpls
        torch.cuda.empty_cache()
        best_h = np.empty(ni, dtype=pkg.BEST_DTYPE)

        def e2e_step():
            plan.load_images(imgs_h, stream=stream)
            plan.load_templates(tpls_h, stream=stream)
            if world > 1:
                b = pkg.distributed_align(plan, stream=stream)
                best_h[:] = pkg.best_to_numpy(b)
            else:
                best_h[:] = plan.align_host(stream=stream)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": total_ips * args.steps / (e_ms / 1e3), "unit": "inner products/s",
               "h2d_bytes_per_step": int(imgs_h.numel() * 8 + (hi - lo) * cfg.n_k * cfg.n_psi * 8),
               "d2h_bytes_per_step": int(ni * 16), "ms_per_step": e_ms / args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ci, cj = {"tiny": (4, 4), "c2": (32, 64), "c3": (16, 64), "c4": (4, 16), "c5": (8, 32)}[cfg.name]
        src_i = (imgs_h if e2e is not None else imgs)[:ci].cpu().numpy()
        src_j = (tpls_h if e2e is not None else tpls)[:cj].cpu().numpy()
        cpu = cpu_baseline(cfg, src_i, src_j, k)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "inner products/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt_ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "fp16x3" if engine == pkg.ENGINE_TC else "f32", "data": "synthetic",
                "config": {"workload": cfg.name, "n": cfg.n, "K": cfg.K, "n_k": cfg.n_k, "n_psi": cfg.n_psi,
                           "n_gamma": n_gamma,
                           "N_im": ni, "N_tm": nj, "N_t": n_t, "eps": cfg.eps, "H": info["H"],
                           "H_plus": info["H_plus"], "K3": info["K3"], "engine": args.engine,
                           **({"ctf_defoci_A": defoci, "n_tau": len(defoci),
                               "ctf_model": "weak-phase, 300 kV, Cs 2.7 mm, A 0.07, 4 A/px"} if defoci else {}),
                           "parallelism": f"template-shard x{world}", "l2": "inputs (6+ GB FB arrays) exceed L2",
                           "input": (f"pixels {cfg.n}x{cfg.n} float32 (NUFFT front end in the step)" if args.pixels
                                     else "polar Fourier samples complex64 [N][n_k][n_psi]"),
                           "step": "load FFT (images+templates) + Steps 1-3 + argmax (+ all-gather/merge)"
                           if args.marginal_tau <= 0 else
                           f"load FFT + Steps 1-3 + log-marginal epilogue (tau = {args.marginal_tau})"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks,
                "kernel_ms": {k2: v[0] / args.steps for k2, v in kt_acc.items()}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
