"""bench.py — low-rank eps^-1 build time on B200 (BASELINE.json metric).

One step = the factored eps^-1 build, stages 1-5 (ISDF point selection, Theta
fit, Cauchy quadrature of the core, G-space Theta^T V Theta, SMW core K), plus
eps^-1 applied to the seeded 8-column probe block, on the Si64-sized config
(BASELINE.json configs[1], the primary 1-GPU roofline case):

  value      device time per build with inputs resident in HBM (CUDA events
             on the library stream, max over ranks)
  e2e        the same step through the C-ABI from pinned HOST buffers: the
             H2D copy of Phi and of the probe and the D2H of eps^-1 X inside
             the timed region
  roofline   the dominant kernel of the step (largest device-time share),
             algorithmic FLOPs / its CUDA-event duration against
             the measured FP64 peak (profiles/FP64_PEAK.json: DMMA 37.17
             TFLOP/s; MEASURED_PEAKS.json has no FP64 entry)
  cpu_baseline  the reference CPU implementation (oracle/_ref) on the host
             cores on a bounded, extrapolated sample (oracle/cpu_baseline.py)

Inputs are larger than L2 (Phi 226 MB, Theta 906 MB) — no explicit flush.
N > 1 (torchrun): the sharded build (dist.py, --mode sharded, default):
grid-row panels, quadrature nodes split across ranks, NCCL all-reduces and
one all-to-all — strong scaling of one build of the config; --mode replicas
runs one full build per rank instead (weak).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config si64] [--impl ours|reference]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.17  # profiles/FP64_PEAK.json (measured DMMA loop, 148 SMs, 1965 MHz)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm = 6552.3
    if os.path.exists(p):
        try:
            hbm = float(json.load(open(p)).get("hbm_gbs", hbm))
        except Exception:
            pass
    return hbm


def algorithmic_work(cfg, n_mu):
    """Per-launch algorithmic FLOPs / bytes."""
    n_r, n = cfg.n_r, cfg.n_v + cfg.n_c
    nh = (cfg.dims[0] // 2 + 1) * cfg.dims[1] * cfg.dims[2]
    return {
        "select": ("tensor", 2.0 * n_r * (n_mu * n + n_mu * (n_mu - 1) / 2.0)),
        # fused fit (lrgw_build): Theta = L L_P^-1 with L_P^-1 lower triangular
        # -> n_r n_mu^2 / 2 multiply-adds; the unfused lhs pass is skipped
        "fit_gemm": ("tensor", 1.0 * n_r * n_mu * n_mu),
        "contour": ("tensor", 2.0 * n_mu * (n_mu + 1) * n * (cfg.n_lambda + 1)),
        # the K3 kernel alone (CUDA events around its launch; the stage adds the
        # node tables, their upload and the fixed-order segment reduction)
        "quad_kernel": ("tensor", 2.0 * n_mu * (n_mu + 1) * n * (cfg.n_lambda + 1)),
        "fft": ("hbm", 8.0 * n_r * n_mu + 16.0 * nh * n_mu),
        "pvp": ("tensor", 1.0 * n_r * n_mu * (n_mu + 1)),
    }


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, gpu):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        out = self.proc.communicate()[0].strip().splitlines()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(int(float(f[0])))
                mx = max(mx, int(float(f[1])))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        backend = "nccl" if args.impl == "ours" else "gloo"
        dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world, device):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_config(cfg):
    """The config the CPU reference is timed on and the factor to this one:
    Si512 is timed on Si216 and extrapolated by the N^3 model (BASELINE.json
    configs[4]); every other config is sampled directly."""
    from paper_2403_12340_b200 import synth

    if cfg.name == "si512":
        small = synth.CONFIGS["si216"]
        return small, (cfg.n_v / small.n_v) ** 3
    return cfg, 1.0


def run_ours(args, cfg, world, rank, local):
    import torch

    from paper_2403_12340_b200 import lrgw, synth

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = lrgw.Context(local)
    stream = torch.cuda.ExternalStream(lrgw.L.load().lrgw_ctx_stream(ctx.handle), device=dev)
    psi = synth.orbitals_device(cfg, seed=1, device=dev)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # the QR work area (Si512: ~14 GB) back to the device before the builds
    e = synth.energies(cfg)
    phi_v, phi_c = psi[:, :cfg.n_v], psi[:, cfg.n_v:]
    x_host = synth.probe_host(cfg.n_r)
    x_dev = torch.from_numpy(np.ascontiguousarray(x_host.T)).to(dev).t()
    y_dev = torch.empty(8, cfg.n_r, dtype=torch.float64, device=dev).t()
    torch.cuda.synchronize()

    def step_dev():
        ep = lrgw.build(phi_v, phi_c, e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda, ctx=ctx)
        lrgw.eps_apply_dev(ep, x_dev, y_dev)
        return ep

    for _ in range(args.warmup):
        step_dev().close()
    torch.cuda.synchronize()

    # ---- device-resident timed region ----
    barrier(world)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    launches0 = ctx.kernel_launches()
    stage_acc = {}
    t_steps = []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        e0.record(stream)
        ep = step_dev()
        e1.record(stream)
        e1.synchronize()
        t_steps.append(e0.elapsed_time(e1))
        for k, v in ctx.stage_ms().items():
            stage_acc.setdefault(k, []).append(v)
        points = ep.point_indices  # the CPU baseline's fit sample uses the build's own ISDF points
        ep.close()
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    launches = ctx.kernel_launches() - launches0
    ms_local = sum(t_steps) / len(t_steps)
    ms = max_over_ranks(ms_local, world, dev)

    # ---- e2e through the C-ABI from pinned host buffers ----
    psi_h = torch.empty(psi.shape[1], psi.shape[0], dtype=torch.float64).pin_memory()
    psi_h.copy_(psi.t())
    x_h = torch.from_numpy(np.ascontiguousarray(x_host.T)).pin_memory()
    y_h = torch.empty(8, cfg.n_r, dtype=torch.float64).pin_memory()
    psi_d = psi.t()  # the H2D lands in the orbitals' own storage (no second N_r x N_b copy in HBM)
    x_d = torch.empty(8, cfg.n_r, dtype=torch.float64, device=dev)
    y_d = torch.empty(8, cfg.n_r, dtype=torch.float64, device=dev)

    def step_e2e():
        with torch.cuda.stream(stream):
            psi_d.copy_(psi_h, non_blocking=True)
            x_d.copy_(x_h, non_blocking=True)
        pd = psi_d.t()
        ep = lrgw.build(pd[:, :cfg.n_v], pd[:, cfg.n_v:], e, cfg.dims, cfg.cell3, k_mu=cfg.k_mu,
                        n_lambda=cfg.n_lambda, ctx=ctx)
        lrgw.eps_apply_dev(ep, x_d.t(), y_d.t())
        with torch.cuda.stream(stream):
            y_h.copy_(y_d, non_blocking=True)
        ep.close()

    step_e2e()
    torch.cuda.synchronize()
    barrier(world)
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 5))):
        e0.record(stream)
        step_e2e()
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    e2e = max_over_ranks(sum(e2e_ms) / len(e2e_ms), world, dev)
    h2d = psi_h.numel() * 8 + x_h.numel() * 8
    d2h = y_h.numel() * 8
    # parity guard on the bench output: eps^-1 X finite and the probe changed
    assert torch.isfinite(y_d).all()

    stages = {k: statistics.median(v) for k, v in stage_acc.items()}
    n_mu = min(max(lrgw.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c), 1), cfg.n_r)
    work = algorithmic_work(cfg, n_mu)
    hbm = _peaks()
    kernels = {}
    for k, (bound, amount) in work.items():
        t = stages.get(k, 0.0)
        if t <= 0:
            continue
        if bound == "tensor":
            ach = amount / (t * 1e-3) / 1e12
            kernels[k] = {"ms": round(t, 4), "bound": "tensor", "achieved": round(ach, 3),
                          "unit": "TFLOP/s", "frac": round(ach / FP64_PEAK_TFLOPS, 4)}
        else:
            ach = amount / (t * 1e-3) / 1e9
            kernels[k] = {"ms": round(t, 4), "bound": "hbm", "achieved": round(ach, 1), "unit": "GB/s",
                          "frac": round(ach / hbm, 4)}
    for k in ("fit_solve", "smw"):
        kernels[k] = {"ms": round(stages.get(k, 0.0), 4), "bound": "latency (N_mu^3 leaves)"}
    kernels["select"]["note"] = "stage of ~18 launches per candidate block (one block per <= 128 pivots), not one kernel"
    # roofline: the dominant single kernel (stages whose events bracket one
    # launch: the Theta^T V Theta SYRK, the fit GEMM, the K3 quadrature kernel)
    dom = max(("pvp", "fit_gemm", "quad_kernel"), key=lambda k: kernels.get(k, {}).get("ms", -1.0))
    dk = kernels[dom]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_r01.json")
    if os.path.exists(tp) and cfg.name == "si64":  # the committed ncu traffic capture is of the Si64 build
        traffic = json.load(open(tp)).get(dom)
    roofline = {"kernel": dom, "bound": dk["bound"], "achieved": dk["achieved"],
                "peak": FP64_PEAK_TFLOPS if dk["bound"] == "tensor" else hbm,
                "unit": dk["unit"], "frac": dk["frac"], "traffic": traffic,
                "peak_source": "profiles/FP64_PEAK.json (measured DMMA)" if dk["bound"] == "tensor"
                else "MEASURED_PEAKS.json hbm_gbs"}
    return {"ms": ms, "e2e_ms": e2e, "h2d": h2d, "d2h": d2h, "launches": launches, "clocks": clk,
            "stages": stages, "kernels": kernels, "roofline": roofline, "psi": psi, "e": e, "ctx": ctx,
            "points": points}


def run_sharded(args, cfg, world, rank, local):
    """The multi-rank build (paper_2403_12340_b200/dist.py + the device
    backend): grid-row panels for selection / fit / the slab FFT, quadrature
    nodes split across ranks, NCCL all-reduces of the N_mu^2 partials and one
    all-to-all of the slab spectra. Strong scaling: one build of the config
    across all ranks; CUDA events on each rank, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2403_12340_b200 import dist as D
    from paper_2403_12340_b200 import lrgw, synth
    from paper_2403_12340_b200.dist_cuda import CudaBackend

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    comm = D.Comm()
    psi = synth.orbitals_device(cfg, seed=1, device=dev)
    e = synth.energies(cfg)
    x_host = synth.probe_host(cfg.n_r)
    n_mu = lrgw.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c)
    ctx = lrgw.Context(local)
    r0, r1 = D.z_panels(cfg.dims, world)[rank]
    # this rank's panel of Phi (column-major) and of the probe, host-pinned for e2e
    psi_p = psi[r0:r1].t().contiguous().t()
    del psi
    psi_h = torch.empty(psi_p.shape[1], psi_p.shape[0], dtype=torch.float64).pin_memory()
    psi_h.copy_(psi_p.t())
    x_p = np.ascontiguousarray(x_host[r0:r1])

    def step(phi_p):
        b = D.DistributedBuild(comm, CudaBackend(n_mu, ctx), cfg.dims, cfg.cell3, cfg.n_v, cfg.n_c, k_mu=cfg.k_mu,
                               n_lambda=cfg.n_lambda, batch=128)
        a, bb = phi_p[:, :cfg.n_v], phi_p[:, cfg.n_v:]
        pts = b.select(a, bb)
        b.fit(pts)
        pv, pc = b.point_rows(pts, a, bb)
        t = b.contour(pv, pc, e)
        k = b.smw(t, b.pvp())
        return b.apply(k, x_p)

    for _ in range(args.warmup):
        step(psi_p)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = Clocks(local)
    launches0 = ctx.kernel_launches()
    t_steps = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        y = step(psi_p)
        e1.record()
        e1.synchronize()
        t_steps.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = ctx.kernel_launches() - launches0
    assert np.isfinite(y).all()
    ms = max_over_ranks(sum(t_steps) / len(t_steps), world, dev)
    # e2e: the panel H2D from pinned host inside the timed region (the probe
    # panel enters and eps^-1 x leaves through the host in apply)
    psi_d = torch.empty_like(psi_h, device=dev)
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        psi_d.copy_(psi_h, non_blocking=True)
        y = step(psi_d.t())
        e1.record()
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    e2e = max_over_ranks(sum(e2e_ms) / len(e2e_ms), world, dev)
    h2d = psi_h.numel() * 8 + x_p.size * 8
    d2h = y.size * 8
    return {"ms": ms, "e2e_ms": e2e, "h2d": h2d, "d2h": d2h, "launches": launches, "clocks": clk}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="si64")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default=None, choices=["single", "sharded", "replicas"],
                    help="single (N = 1 default): the one-GPU build; sharded (N > 1 default): one build "
                         "split across the ranks (strong scaling); replicas: one full build per rank")
    args = ap.parse_args()

    from paper_2403_12340_b200 import synth

    cfg = synth.CONFIGS[args.config]
    world, rank, local = dist_setup(args)
    mode = args.mode or ("single" if world == 1 else "sharded")
    if mode == "single" and world > 1:
        mode = "replicas"
    workload = {"workload": f"{cfg.name}: grid {cfg.dims[0]}^3 = {cfg.n_r} points, cell {cfg.cell} bohr, "
                            f"N_v = N_c = {cfg.n_v}, N_mu = {int(round(cfg.k_mu * (cfg.n_v * cfg.n_c) ** 0.5))}, "
                            f"N_lambda = {cfg.n_lambda}, eps^-1 X on an {cfg.n_r}x8 probe",
                "stages": "1-5 (select, fit, quadrature, Coulomb/ThetaVTheta, SMW) + probe apply",
                "l2": f"inputs larger than L2 (Phi {cfg.n_r * (cfg.n_v + cfg.n_c) * 8 / 1e6:.0f} MB, Theta "
                      f"{cfg.n_r * int(round(cfg.k_mu * (cfg.n_v * cfg.n_c) ** 0.5)) * 8 / 1e6:.0f} MB); no flush",
                "parallelism": {"single": "1 GPU", "replicas": f"replicas x{world}",
                                "sharded": f"sharded x{world} (grid-row panels, node split, NCCL)"}[mode]}
    metric = "low-rank eps^-1 build time (s), stages 1-5 + probe apply"

    if args.impl == "reference":
        if rank != 0:
            return
        from oracle import cpu_baseline

        cores = os.cpu_count() or 1
        vals = []
        ccfg, scale = cpu_config(cfg)
        for i in range(args.warmup + args.steps):  # W untimed warm-up samples, then K timed
            r = cpu_baseline.run(ccfg, cores=cores, sel_steps=16, fit_rows=(1536, 2560), cols=64, seed=5 + i)
            if i >= args.warmup:
                vals.append(r["total_s"] * scale)
        if scale != 1.0:
            r["sample"] += f"; x{scale:.2f} = (N_v {cfg.n_v} / {ccfg.n_v})^3 (N^3 model, BASELINE.json configs[4])"
            r["stages"] = {k: v * scale for k, v in r["stages"].items()}
        v = statistics.median(vals)
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
                "config": workload,
                "cpu_baseline": {"value": v, "unit": "s", "cores": r["cores"], "kind": "reference",
                                 "sample": r["sample"], "stages_s": r["stages"],
                                 "no_select_s": statistics.median(vals) - r["stages"]["select"]},
                "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    if mode == "sharded":
        res = run_sharded(args, cfg, world, rank, local)
        if rank == 0:
            line = {"metric": metric, "value": res["ms"] / 1e3, "unit": "s", "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms"],
                    "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                    "data": "synthetic (seeded)", "config": workload,
                    "e2e": {"value": res["e2e_ms"] / 1e3, "unit": "s", "h2d_bytes_per_step": res["h2d"],
                            "d2h_bytes_per_step": res["d2h"]},
                    "gpu_launches": res["launches"], "clocks": res["clocks"], "roofline": None,
                    "cpu_baseline": None}
            print(json.dumps(line))
        import torch.distributed as dist

        dist.destroy_process_group()
        return
    res = run_ours(args, cfg, world, rank, local)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import cpu_baseline

        ccfg, scale = cpu_config(cfg)
        if ccfg is cfg:
            psi_h = np.asfortranarray(res["psi"].cpu().numpy())
            r = cpu_baseline.run(cfg, psi=psi_h, energies=res["e"], cores=os.cpu_count(), points=res["points"])
        else:
            r = cpu_baseline.run(ccfg, cores=os.cpu_count())
        cpu = {"value": r["total_s"] * scale, "unit": "s", "cores": r["cores"], "kind": "reference",
               "sample": r["sample"] + (f"; then x{scale:.2f} = (N_v {cfg.n_v} / {ccfg.n_v})^3, the N^3 model of "
                                        f"BASELINE.json configs[4] (extrapolated, not run at {cfg.name})"
                                        if scale != 1.0 else ""),
               "stages_s": {k: round(v * scale, 3) for k, v in r["stages"].items()},
               "no_select_s": r["total_no_select_s"] * scale}
    if rank == 0:
        line = {"metric": metric, "value": res["ms"] / 1e3, "unit": "s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms"], "higher_is_better": False,
                "scaling": "weak" if mode == "replicas" else "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded)", "config": workload,
                "e2e": {"value": res["e2e_ms"] / 1e3, "unit": "s", "h2d_bytes_per_step": res["h2d"],
                        "d2h_bytes_per_step": res["d2h"]},
                "gpu_launches": res["launches"], "clocks": res["clocks"],
                "roofline": res["roofline"], "stages_ms": {k: round(v, 4) for k, v in res["stages"].items()},
                "kernels": res["kernels"], "cpu_baseline": cpu}
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
