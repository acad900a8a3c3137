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
    on a bounded slab sample of the same workload, extrapolated linearly in J.
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
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------------------------
# CPU reference arm (oracle = call-for-call restatement of cpfast, bounded slab sample)
# ----------------------------------------------------------------------------------------------
def cpu_sample_config(cfg):
    """Bounded sample of the workload: same dims except the last mode, cut so that one reference
    iteration takes O(1-5) s on the host (the reference needs ~4x the tensor in RAM)."""
    from paper_1205_2584_b200 import synth

    j = int(np.prod(cfg.dims))
    target = 1.25e8  # elements (1 GB fp64)
    if j <= target:
        return cfg, 1.0
    last = max(1, int(cfg.dims[-1] * target / j))
    small = synth.scaled(cfg, tuple(cfg.dims[:-1]) + (last,), name=cfg.name + "_sample")
    return small, j / float(np.prod(small.dims))


def fast_tensor(cfg, seed):
    """Sample tensor for the CPU timing (BLAS path is fine here: timing, not parity)."""
    from paper_1205_2584_b200 import synth

    fac = synth.truth_factors(cfg, seed) if np.prod(cfg.dims) < 2e7 else None
    rng = np.random.default_rng([seed, 100])
    if fac is None:
        fac = []
        for d in cfg.dims:
            q, _ = np.linalg.qr(rng.standard_normal((d, cfg.rank)))
            fac.append(q)
    kr = fac[0]
    for f in fac[1:-1]:
        kr = (f[:, None, :] * kr[None, :, :]).reshape(-1, cfg.rank)
    x = (kr @ fac[-1].T).reshape(tuple(cfg.dims), order="F")
    sigma = np.linalg.norm(x) / math.sqrt(x.size * 10.0 ** (cfg.snr_db / 10.0))
    x += sigma * np.random.default_rng([seed, 1]).standard_normal(x.shape)
    return np.asfortranarray(x)


def run_cpu_reference(cfg, seed, iters, warmup=1):
    """Time `iters` reference iterations (after `warmup`) on a sample; returns it/s at full size."""
    from oracle import cp_oracle
    from paper_1205_2584_b200 import synth

    small, scale = cpu_sample_config(cfg)
    y = fast_tensor(small, seed)
    stamps = {}

    def on_iter(t):
        stamps[t] = time.perf_counter()

    conf = cp_oracle.OracleConfig(rank=small.rank, tau=synth.tau_for_unit_mu(small, seed), tol=0.0,
                                  max_iters=warmup + iters, seed=seed)
    cp_oracle.fit_lm(y, conf, on_iter=on_iter)
    dt = stamps[warmup + iters] - stamps[warmup]
    per_sample = iters / dt
    desc = (f"reference fLM (oracle/cp_oracle.py, bit-exact restatement of cpfast) on a "
            f"{'x'.join(map(str, small.dims))} slab of the {'x'.join(map(str, cfg.dims))} tensor, R={cfg.rank}, "
            f"{iters} timed iterations after {warmup} warm-up; it/s extrapolated x{scale:.2f} (linear in J)")
    return per_sample / scale, desc, os.cpu_count()


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
        iters = max(1, min(args.steps, 3))
        v, desc, cores = run_cpu_reference(cfg, args.seed, iters, warmup=min(args.warmup, 1))
        line({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
              "steps": iters, "warmup": min(args.warmup, 1), "ms_per_step": 1e3 / v, "higher_is_better": True,
              "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
              "config": config_desc,
              "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc},
              "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
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
    y_dev = synth.device_tensor(cfg, args.seed, device=f"cuda:{local}", slab=(lo, hi))
    torch.cuda.synchronize()
    ctx = _Dist() if world > 1 else None
    uid = ctx.unique_id() if ctx else None
    eng = _native.Engine(kind, cfg.dims, cfg.rank, local, rank, world, uid)
    eng.set_tensor_device(y_dev.data_ptr(), y_dev.numel())
    init = np.concatenate([f.reshape(-1, order="F") for f in synth.init_factors(cfg, args.seed)])
    eng.set_factors(init)
    tau = synth.tau_for_unit_mu(cfg, args.seed)
    K, W = args.steps, args.warmup
    NP = 3  # extra eagerly-launched, event-profiled iterations for the per-phase roofline numbers
    eng.fit_begin("auto", tau, 0.0, W + K + NP)
    eng.fit_step(W)  # warm-up (also captures the per-iteration CUDA graph)
    stream = torch.cuda.ExternalStream(eng.stream_handle)
    launches0 = eng.launch_count()
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    st = eng.fit_step(K)
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    iters_done = st.iter - W
    launches = eng.launch_count() - launches0
    # per-phase device times from CUDA events on the engine stream (eager launches)
    eng.profile(True)
    ms0, cnt0 = eng.phase_times()
    st2 = eng.fit_step(NP)
    ms1, cnt1 = eng.phase_times()
    eng.profile(False)
    np_done = max(st2.iter - st.iter, 1)
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = iters_done / (ms / 1e3)

    # roofline of pass A (every-iteration tensor pass)
    pk, pk_kind = peaks()
    na = cnt1[0] - cnt0[0]
    t_a = (ms1[0] - ms0[0]) / max(na, 1)
    bytes_a = (hi - lo) * int(np.prod(cfg.dims[:-1])) * esize
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
                                 "tensor cores, exact 8-digit split of the fp64 operands (tcgen05 kind::i8)",
             _native.PASS_DMMA: "k_pass_dmma<NT,0>: pass A (MTTKRP modes 1..N-1 + trial-fit contraction) on the "
                                "fp64 tensor cores (DMMA)",
             _native.PASS_FMA: "k_pass_a2: pass A (MTTKRP modes 1..N-1 + trial-fit contraction), fp64 FMA"}[impl]
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": traffic,
                "kernel": kname,
                "bytes_per_launch": bytes_a, "avg_launch_ms": round(t_a, 4), "launches": na,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})",
                "share_of_step": round(((ms1[0] - ms0[0]) / np_done) / (ms / max(iters_done, 1)), 4) if ms > 0 else None,
                "phase_ms_per_step": {k: round((ms1[i] - ms0[i]) / np_done, 4)
                                      for i, k in enumerate(["pass_a", "pass_b", "lu", "solve"])},
                "phase_note": f"CUDA events around each phase over {np_done} eagerly launched iterations after the timed region"}
    eng.close()

    # end-to-end through the public API, tensor in pinned host memory
    e2e = None
    if not args.no_e2e:
        host = torch.empty(y_dev.shape, dtype=y_dev.dtype, pin_memory=True)
        host.copy_(y_dev)
        del y_dev
        torch.cuda.empty_cache()
        arr = host.numpy()
        local_dims = tuple(cfg.dims[:-1]) + (hi - lo,)
        y_host = np.reshape(arr.T, local_dims, order="F")
        conf = FitConfig(rank=cfg.rank, variant="auto", tau=tau, tol=0.0, max_iters=K, seed=args.seed, init="random")
        # process setup, untimed: grow the engine memory pool to the fit's footprint (tensor copy +
        # digit-plane images + workspace), so the timed call reuses memory instead of mapping it
        _native.pool_reserve(local, 4 * y_host.nbytes + (2 << 30))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        res = fit(y_host, conf, device=local, distributed=ctx, slab_of=cfg.dims[-1])
        t1 = time.perf_counter()
        wall = t1 - t0
        if dist:
            t = torch.tensor([wall], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall = float(t.item())
        rt = cfg.rank * sum(cfg.dims)
        e2e = {"value": res.iters / wall, "unit": UNIT,
               "h2d_bytes_per_step": int(y_host.nbytes // max(res.iters, 1)),
               "d2h_bytes_per_step": int(rt * esize // max(res.iters, 1)),
               "what": "public fit() from pinned host memory: H2D of the tensor slab, preamble, "
                       f"{res.iters} iterations, factor download; wall clock max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, desc, cores = run_cpu_reference(cfg, args.seed, 2, warmup=1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc}

    if rank == 0:
        line({"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": iters_done,
              "warmup": W, "ms_per_step": round(ms / max(iters_done, 1), 4), "higher_is_better": True,
              "scaling": "strong", "vs_baseline": None, "dtype": "f64" if not cfg.complex_ else "c128",
              "data": "synthetic (seeded congruence construction, SURVEY App. B; device-generated)",
              "config": config_desc, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
              "cpu_baseline": cpu, "clocks": clocks,
              "accepted_in_timed": None})
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
