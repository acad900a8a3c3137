"""Throughput benchmark: fast damped Gauss-Newton (fLM) iterations/sec on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl b200|reference]

Contract:
  * a step = one fLM iteration (candidate + trial fit + accept/commit) over the whole tensor;
  * workload = BASELINE config 4 (1000x1000x2000 fp64, R=20, 16 GB) unless --config says
    otherwise; the tensor is slab-sharded along mode 3 across N GPUs (torchrun, one rank per
    GPU, NCCL), so the total work is fixed as N grows ("scaling": "strong");
  * value = K / (max over ranks of the device time of K iterations), timed with CUDA events
    on the engine's stream with barrier + synchronize on both sides, inputs resident in HBM;
    the 16 GB tensor is larger than the 126 MB L2, so no flush is needed between iterations;
  * e2e = the same metric through the public drop-in ``fit()`` with the tensor in pinned HOST
    memory (H2D upload, preamble, K iterations, factor download inside the timed region);
  * roofline = pass A (the every-iteration MTTKRP/trial-fit tensor pass), algorithmic bytes
    J_local * 8 per launch over its CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs;
  * cpu_baseline / --impl reference = the reference algorithm (oracle/cp_oracle.py, a call-for-
    call NumPy restatement of cpfast pinned bit-exact against the reference) on the host cores,
    on a bounded sample of the same construction (1000x1000x32 at config 4), the same iteration
    window as the GPU arm; its tensor-sized time is scaled by J_full / J_sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fast-dGN iterations/sec (fp64)"
UNIT = "iterations/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c4")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 20 ms around the timed region.  nvidia-smi
    needs ~0.5 s to start, longer than a 20-step timed region, so the sampler is started first and
    the timed region begins once it is producing rows; rows are stamped with the host clock when
    read, and the ones inside [begin, end] of the timed region (widened by one sampling period)
    are the reported samples (``samples_in_window``)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 20

    def __init__(self, index: int):
        import threading

        self.rows = []
        self.t_begin = self.t_end = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
        except Exception:
            self.p = None
            return
        self.th = threading.Thread(target=self._reader, daemon=True)
        self.th.start()
        t0 = time.perf_counter()
        while not self.rows and time.perf_counter() - t0 < 10.0 and self.p.poll() is None:
            time.sleep(0.01)

    def _reader(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.perf_counter(), parts))

    def begin(self):
        self.t_begin = time.perf_counter()

    def end(self):
        self.t_end = time.perf_counter()
        time.sleep(2.5 * self.PERIOD_MS / 1e3)  # let the row covering the region's end arrive

    def stop(self):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.th.join(timeout=2)
        rows = [r for _, r in self.rows]
        if self.t_begin is not None and self.t_end is not None:
            pad = 1.5 * self.PERIOD_MS / 1e3
            win = [r for t, r in self.rows if self.t_begin - pad <= t <= self.t_end + pad]
        else:
            win = rows
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0,
                    "samples_in_window": 0, "samples_total": len(rows)}
        sm = [float(r[0]) for r in win if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in win for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(win[0][1]),
                "reasons": reasons, "samples": len(win), "samples_in_window": len(win),
                "samples_total": len(rows), "period_ms": self.PERIOD_MS}


# ----------------------------------------------------------------------------------------------
# CPU reference arm (oracle = call-for-call restatement of cpfast, bounded slab sample)
# ----------------------------------------------------------------------------------------------
SAMPLE_ELEMS = 3.2e7   # ~256 MB fp64: one reference iteration is O(1 s) on the host, the whole
                       # --steps/--warmup run a few minutes; the full config-4 tensor would need
                       # ~63 GB of host RAM in the reference and ~30-300 s per iteration


def host_info() -> dict:
    """What the CPU numbers ran on: cores, affinity, cgroup quota, RAM, BLAS threads."""
    info = {"nproc": os.cpu_count()}
    try:
        info["affinity_cpus"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    try:
        q = Path("/sys/fs/cgroup/cpu.max").read_text().split()
        info["cgroup_cpu_max"] = None if q[0] == "max" else round(int(q[0]) / int(q[1]), 2)
    except Exception:
        pass
    try:
        mem = {ln.split(":")[0]: int(ln.split()[1]) for ln in Path("/proc/meminfo").read_text().splitlines()
               if ln.startswith(("MemTotal", "MemAvailable"))}
        info["ram_total_gb"] = round(mem["MemTotal"] / 2**20, 1)
        info["ram_available_gb"] = round(mem["MemAvailable"] / 2**20, 1)
    except Exception:
        pass
    try:
        from threadpoolctl import threadpool_info

        info["blas"] = [{k: d.get(k) for k in ("internal_api", "version", "num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    info["OPENBLAS_NUM_THREADS"] = os.environ.get("OPENBLAS_NUM_THREADS")
    return info


def cpu_sample_config(cfg):
    """Bounded sample of the workload: the same construction (synth.make_tensor) with
    the last mode cut so the sample has ~SAMPLE_ELEMS elements."""
    from paper_1205_2584_b200 import synth

    j = int(np.prod(cfg.dims))
    if j <= SAMPLE_ELEMS:
        return cfg, 1.0
    last = max(1, int(math.ceil(cfg.dims[-1] * SAMPLE_ELEMS / j)))
    small = synth.scaled(cfg, tuple(cfg.dims[:-1]) + (last,), name=cfg.name + "_sample")
    return small, j / float(np.prod(small.dims))


def run_cpu_reference(cfg, seed, steps, warmup):
    """The reference fLM loop (oracle port) for warmup + steps iterations on the sample -- the same
    iteration window as the GPU arm.  Per iteration the oracle reports the J-independent time (fLM
    candidate incl. the NR^2 core inverse, gradient, decision) and the tensor-sized time (trial
    relative error, and the N MTTKRPs of an accepted step); the full-size estimate scales only the
    latter by J_full / J_sample."""
    from oracle import cp_oracle
    from paper_1205_2584_b200 import synth

    small, scale = cpu_sample_config(cfg)
    y = synth.make_tensor(small, seed)
    stamps, phases = {}, []

    def on_iter(t):
        stamps[t] = time.perf_counter()

    conf = cp_oracle.OracleConfig(rank=small.rank, tau=synth.tau_for_unit_mu(small, seed), tol=0.0,
                                  max_iters=warmup + steps, seed=seed)
    res = cp_oracle.fit_lm(y, conf, on_iter=on_iter, phases=phases)
    timed = phases[warmup:warmup + steps]
    sample_s = stamps[warmup + steps] - stamps[warmup]
    core_s = sum(p[0] for p in timed)
    tensor_s = sum(p[1] for p in timed)
    full_s = core_s + scale * tensor_s
    accepted = sum(1 for t in res.trace[warmup:warmup + steps] if t[3])
    sample = (f"reference fLM (oracle/cp_oracle.py, bit-exact restatement of cpfast, pinned to cpfast goldens) on "
              f"{'x'.join(map(str, small.dims))} (same construction as {'x'.join(map(str, cfg.dims))}), R={cfg.rank}, "
              f"iterations {warmup + 1}..{warmup + steps} timed after {warmup} warm-up"
              + (f"; full size = J-independent time + {scale:.2f} x tensor-sized time" if scale != 1.0 else ""))
    return {"value": steps / full_s, "ms_per_step": 1e3 * sample_s / steps, "sample_it_s": steps / sample_s,
            "scale_J": scale, "core_ms_per_step": 1e3 * core_s / steps, "tensor_ms_per_step": 1e3 * tensor_s / steps,
            "accepted": accepted, "steps": steps, "warmup": warmup, "sample": sample,
            "cores": os.cpu_count(), "host": host_info()}


def line(d):
    print(json.dumps(d), flush=True)


# ----------------------------------------------------------------------------------------------
def main():
    args = parse()
    from paper_1205_2584_b200 import synth

    cfg = synth.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    config_desc = {"workload": f"BASELINE config {args.config[1:]}: {'x'.join(map(str, cfg.dims))} "
                               f"{'complex128' if cfg.complex_ else 'fp64'} R={cfg.rank}, c={cfg.congruence}, "
                               f"SNR {cfg.snr_db:g} dB, variant auto, tol 0",
                   "global_batch": int(np.prod(cfg.dims)), "seq_len": None,
                   "parallelism": f"slab{world} (mode-{len(cfg.dims)} shards, NCCL allreduce/allgather)",
                   "l2": "no flush: tensor >> 126 MB L2" if np.prod(cfg.dims) * 8 > 126e6 else "L2-resident tensor"}

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_cpu_reference(cfg, args.seed, args.steps, args.warmup)
        extrap = {"sample_value": r["sample_it_s"], "scale_J": r["scale_J"],
                  "core_ms_per_step": r["core_ms_per_step"], "tensor_ms_per_step": r["tensor_ms_per_step"],
                  "model": "full-size it/s = K / (sum of J-independent time + scale_J * sum of tensor-sized time)",
                  "why": "the full config-4 tensor needs ~63 GB of host RAM in the reference (4x the tensor) and "
                         "~30-300 s per iteration; the host record shows the RAM"}
        line({"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
              "scaling": "strong", "vs_baseline": None, "dtype": "f64" if not cfg.complex_ else "c128",
              "data": "synthetic", "config": config_desc,
              "value_is": "extrapolated to the full config from the measured sample (ms_per_step is the sample's)"
                          if r["scale_J"] != 1.0 else "measured",
              "extrapolation": extrap if r["scale_J"] != 1.0 else None,
              "accepted_in_timed": r["accepted"], "host": r["host"],
              "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port",
                               "sample": r["sample"]},
              "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1205_2584_b200 import _native, build, slab_bounds
    from paper_1205_2584_b200.solver import FitConfig, _Dist, fit

    if rank == 0:
        build.build()
    if dist:
        dist.barrier()
    _native.load()
    lo, hi = slab_bounds(cfg.dims[-1], world, rank)
    kind = _native.CPF_COMPLEX if cfg.complex_ else _native.CPF_REAL
    esize = 16 if cfg.complex_ else 8
    rt = cfg.rank * sum(cfg.dims)
    y_dev = synth.device_tensor(cfg, args.seed, device=f"cuda:{local}", slab=(lo, hi))
    torch.cuda.synchronize()
    ctx = _Dist() if world > 1 else None
    tau = synth.tau_for_unit_mu(cfg, args.seed)
    K, W = args.steps, args.warmup

    # ---- end to end through the public API, tensor in pinned HOST memory.  Run first, in a fresh
    # process: the cold call allocates the fit's ~50 GB (tensor + int8 images, cudaMalloc); the warm
    # call (after the device-resident timing) is a long-lived process's fit(), reusing the buffers
    # an earlier engine parked in the engine's buffer cache.
    y_host = None
    e2e_runs = {}

    def run_e2e(tag):
        conf = FitConfig(rank=cfg.rank, variant="auto", tau=tau, tol=0.0, max_iters=K, seed=args.seed, init="random")
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        res = fit(y_host, conf, device=local, distributed=ctx, slab_of=cfg.dims[-1])
        wall = time.perf_counter() - t0
        if dist:
            t = torch.tensor([wall], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall = float(t.item())
        e2e_runs[tag] = (res.iters / wall, res)

    if not args.no_e2e:
        host = torch.empty(y_dev.shape, dtype=y_dev.dtype, pin_memory=True)
        host.copy_(y_dev)
        torch.cuda.synchronize()
        local_dims = tuple(cfg.dims[:-1]) + (hi - lo,)
        y_host = np.reshape(host.numpy().T, local_dims, order="F")
        run_e2e("cold")

    # ---- device-resident throughput
    uid = ctx.unique_id() if ctx else None
    eng = _native.Engine(kind, cfg.dims, cfg.rank, local, rank, world, uid)
    eng.set_tensor_device(y_dev.data_ptr(), y_dev.numel())
    init = np.concatenate([f.reshape(-1, order="F") for f in synth.init_factors(cfg, args.seed)])
    eng.set_factors(init)
    NP = 3  # extra eagerly-launched, event-profiled iterations for the per-phase roofline numbers
    # + 1: the fit's last iteration skips the next step's core system, so it is not profiled
    eng.fit_begin("auto", tau, 0.0, W + K + NP + 1)
    eng.fit_step(W)  # warm-up (also captures the per-iteration CUDA graph)
    stream = torch.cuda.ExternalStream(eng.stream_handle)
    launches0 = eng.launch_count()
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler.begin()
    ev0.record(stream)
    st = eng.fit_step(K)
    ev1.record(stream)
    torch.cuda.synchronize()
    sampler.end()
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    iters_done = st.iter - W
    launches = eng.launch_count() - launches0
    trace = eng.trace(W + K)
    accepted = sum(1 for t in trace[W:W + K] if t[3])
    fallbacks, guarded = eng.pass_guard()
    # per-phase device times from CUDA events on the engine stream (eager launches)
    eng.profile(True)
    ms0, cnt0 = eng.phase_times()
    st2 = eng.fit_step(NP)
    ms1, cnt1 = eng.phase_times()
    ph_max = eng.phase_max()
    eng.profile(False)
    np_done = max(st2.iter - st.iter, 1)
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = iters_done / (ms / 1e3)
    ms_step = ms / max(iters_done, 1)

    # roofline of pass A (every-iteration tensor pass)
    pk, pk_kind = peaks()
    na = cnt1[0] - cnt0[0]
    t_a = (ms1[0] - ms0[0]) / max(na, 1)
    j_local = (hi - lo) * int(np.prod(cfg.dims[:-1]))
    bytes_a = j_local * esize
    achieved = bytes_a / (t_a * 1e-3) / 1e9 if t_a > 0 else 0.0
    traffic = None
    prof_json = ROOT / "profiles" / "pass_a_traffic.json"
    if prof_json.exists():
        try:
            traffic = json.loads(prof_json.read_text()).get(args.config)
        except Exception:
            traffic = None
    impl = eng.pass_impl()
    kname = {_native.PASS_OZAKI: "k_oz_pass<0>: pass A (MTTKRP modes 1..N-1 + trial-fit contraction) on the int8 "
                                 "tensor cores, 8-plane digit split of the fp64 operands (Ozaki scheme, tcgen05 "
                                 "kind::i8; accuracy-guarded, fp64 fallback)",
             _native.PASS_DMMA: "k_pass_dmma<NT,0>: pass A (MTTKRP modes 1..N-1 + trial-fit contraction) on the "
                                "fp64 tensor cores (DMMA)",
             _native.PASS_FMA: "k_pass_a2: pass A (MTTKRP modes 1..N-1 + trial-fit contraction), fp64 FMA"}[impl]
    phase_ms = {k: round((ms1[i] - ms0[i]) / np_done, 4) for i, k in enumerate(["pass_a", "pass_b", "lu", "solve"])}
    # one complete factorisation (+ inverse): the longest LU instance of the profiled iterations --
    # the per-step total also holds gated instances (a rejected step skips the fork's, an accepted
    # step abandons the speculated one) and, with the speculative branch, two per step
    lu_one = round(ph_max[2], 4) if ph_max[2] > 0 else phase_ms["lu"]
    # core system: LU with partial pivoting (2/3 n^3) + the explicit inverse of both triangles
    # (2/3 n^3) when the engine forms it (n_B <= 2560), once per iteration; solves: 3 B-applications
    # of 2 triangular mat-vecs (2 n^2 flop each) -- real flops, x4 for complex
    n_b = len(cfg.dims) * cfg.rank ** 2
    cw = 4.0 if cfg.complex_ else 1.0
    inv = n_b <= 2560
    lu_flops = cw * ((2.0 / 3.0) + ((2.0 / 3.0) if inv else 0.0)) * n_b ** 3
    solve_flops = cw * 3 * 2 * 2.0 * n_b ** 2
    fp64 = {"dmma_tflops": 37.2, "source": "profiles/r01_fp64_peaks.json (tools/microbench/fp64_peaks.cu)"}
    try:
        fp64 = {"dmma_tflops": json.loads((ROOT / "profiles" / "r01_fp64_peaks.json").read_text())["dmma_tflops"],
                "source": fp64["source"]}
    except Exception:
        pass
    step_bytes = j_local * esize * (1.0 + accepted / max(iters_done, 1))
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": traffic,
                "kernel": kname,
                "bytes_per_launch": bytes_a, "avg_launch_ms": round(t_a, 4), "launches": na,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})",
                "share_of_step": round(((ms1[0] - ms0[0]) / np_done) / ms_step, 4) if ms > 0 else None,
                "phase_ms_per_step": phase_ms,
                "phase_note": f"CUDA events around each phase over {np_done} eagerly launched iterations after the timed region; "
                              "lu = all core-system factorisations of a step (the fork's and the speculated one's, "
                              "some gated off), phases.lu.ms_per_factorisation = one complete factorisation as it "
                              "runs in the step (beside the tensor pass)",
                "phases": {
                    "lu": {"bound": "fp64 (DMMA)", "n_B": n_b, "flop_per_factorisation": lu_flops,
                           "what": "LU with partial pivoting of Phi" + (" + explicit inv(L), inv(U)" if inv else ""),
                           "ms_per_factorisation": lu_one,
                           "achieved_tflops": round(lu_flops / (lu_one * 1e-3) / 1e12, 3) if lu_one > 0 else None,
                           "peak_tflops": fp64["dmma_tflops"], "peak_source": fp64["source"],
                           "frac": round(lu_flops / (lu_one * 1e-3) / 1e12 / fp64["dmma_tflops"], 4) if lu_one > 0 else None},
                    "solve": {"bound": "L2 (Phi^-1 resident)", "flop_per_step": solve_flops,
                              "achieved_tflops": round(solve_flops / (phase_ms["solve"] * 1e-3) / 1e12, 4) if phase_ms["solve"] > 0 else None,
                              "frac": round(solve_flops / (phase_ms["solve"] * 1e-3) / 1e12 / fp64["dmma_tflops"], 5) if phase_ms["solve"] > 0 else None},
                    "step": {"bound": "hbm", "bytes_per_step": step_bytes,
                             "what": "pass A every step + pass B on accepted steps, J_local * 8 B each",
                             "hbm_bound_ms": round(step_bytes / (pk["hbm_gbs"] * 1e9) * 1e3, 4),
                             "frac": round(step_bytes / (pk["hbm_gbs"] * 1e9) * 1e3 / ms_step, 4)}}}
    eng.close()

    e2e = None
    if not args.no_e2e:
        del y_dev
        torch.cuda.empty_cache()
        run_e2e("warm")
        v_warm, res = e2e_runs["warm"]
        v_cold = e2e_runs["cold"][0]
        e2e = {"value": v_warm, "unit": UNIT,
               "h2d_bytes_per_step": int(y_host.nbytes // max(res.iters, 1)),
               "d2h_bytes_per_step": int(rt * esize // max(res.iters, 1)),
               "cold_value": v_cold,
               "what": "public fit() from pinned host memory: H2D of the tensor slab, preamble, "
                       f"{res.iters} iterations, factor download; wall clock max over ranks.  value: a process "
                       "that has run a fit before (its tensor-sized buffers are reused from the engine's buffer "
                       "cache); cold_value: the first fit() of the process (allocates them inside the call)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r = run_cpu_reference(cfg, args.seed, 3, 1)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port", "sample": r["sample"],
               "sample_value": r["sample_it_s"], "host": r["host"]}

    if rank == 0:
        line({"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": iters_done,
              "warmup": W, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
              "scaling": "strong", "vs_baseline": None, "dtype": "f64" if not cfg.complex_ else "c128",
              "data": "synthetic (seeded congruence construction, SURVEY App. B; device-generated)",
              "config": config_desc, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
              "cpu_baseline": cpu, "clocks": clocks,
              "accepted_in_timed": accepted, "pass_guard": {"fallbacks": fallbacks, "tensor_rejected": guarded}})
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
