#!/usr/bin/env python
"""FastCLIP loss+grad step benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = the per-rank FastCLIP-v3 loss step (trainer.cpp:427-589) at global B = 5120,
d = 512, N = 2.7M-entry u table, synthetic bf16 unit-norm embeddings. N > 1: launched with
torch.distributed.run, one rank per GPU, global batch fixed (strong scaling); per step the
ranks all-gather E and the per-sample scalar payload through NVLink peer memory (NCCL only
for the one-time set-up, or as the fallback when GPUs cannot map each other's memory).

`value` is device-timed (CUDA events around each step, L2 flushed between steps, inputs
resident in HBM), max over ranks; `e2e` times the same step through the public API with
the inputs copied from pinned host memory and the step scalars read back every step.
`--impl reference` times the reference's own CPU implementation (oracle/_ref, the
reference's translation units) on a bounded anchor-slice sample of the same workload.
"""
from __future__ import annotations

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

METRIC = "FastCLIP loss+grad steps/s at global B=5120, d=512 (1/2/4/8 B200); % TC peak"
UNIT = "steps/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), \
            float(p["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        busy = [x for x in sm if x > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(B, d, N, world, rank, n_sets, seed=0):
    from paper_2407_01445_b200 import synthetic as S
    Bl = B // world
    sets = []
    for s in range(n_sets):
        b1, b2 = S.embeddings(B, d, seed + s)
        ids = S.ids(B, N, seed + s)
        lo = rank * Bl
        sets.append((b1[lo:lo + Bl].copy(), b2[lo:lo + Bl].copy(), ids[lo:lo + Bl].copy()))
    return sets


def cpu_reference_step(B, d, N, variant, log, tau=None):
    """ONE full step of the reference's own CPU path (oracle/_ref_fast: engine.cpp, state.cpp, ...
    compiled from the reference sources, -O3) on the box's host cores, timed directly. The
    reference parallelises over data-parallel workers (one std::thread each,
    fabric.cpp:237-258); we run W workers, the largest divisor of B not above nproc, each with
    its full anchor slice (every anchor's loops and the three full S products of its step,
    engine.cpp:159, :83, :185). Nothing is extrapolated: value = 1 / (measured step time)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2407_01445_b200 import synthetic as S
    nproc = os.cpu_count() or 1
    W = max(w for w in range(1, min(nproc, B) + 1) if B % w == 0)
    b1, b2 = S.embeddings(B, d, 0)
    E1 = S.bf16_to_f32(b1).astype(np.float64)
    E2 = S.bf16_to_f32(b2).astype(np.float64)
    ids = S.ids(B, N, 0)
    cfg = O.default_config(variant, N, **({"tau_init": tau} if tau is not None else {}))
    st = O.new_state(cfg)
    t = time.perf_counter()
    O.step(cfg, st, W, E1, E2, ids, 0.6, 1e-14, backend="ref_fast")
    t_step = time.perf_counter() - t
    cpu_model = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    sample = (f"one full reference step (oracle/_ref TUs, -O3) at B={B}, d={d}, N={N} as {W} fabric workers x "
              f"{B // W} anchors on {nproc} host threads ({cpu_model}); timed directly, not extrapolated")
    log(f"[cpu] W={W} full step {t_step:.1f}s")
    return {"value": 1.0 / t_step, "unit": UNIT, "cores": W, "kind": "reference", "sample": sample,
            "step_s": t_step}


def reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cb = cpu_reference_step(args.batch, args.dim, args.n_train, args.variant, lambda m: print(m, file=sys.stderr),
                            tau=args.tau)
    # one full step is the unit of work and it takes tens of seconds on the host: the line reports
    # the ONE step actually timed (steps_requested / warmup_requested are the driver's K / W)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": 1, "warmup": 0, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": 1e3 / cb["value"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args, world),
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def ncu_traffic(phase):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the phase's kernel, from the
    newest committed ncu --set full summary (profiles/<round>_traffic.json); None if absent."""
    import glob
    kern = {"pass1_stats": ("sim_tile_kernel<3>", "sim_tile_kernel<0>"), "pass2_q": ("sim_tile_kernel<1>",),
            "grad_gemm": ("grad_gemm_kernel", "grad_gemm_kernel<1>"),
            "tables_tau": ("fc_anchor_kernel",)}.get(phase, ())
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "*_traffic.json")))
    if not files:
        return None
    try:
        tab = json.load(open(files[-1]))["bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None
    for k in kern:
        if k in tab:
            return {"bytes": tab[k], "kernel": k, "source": os.path.relpath(files[-1], os.path.dirname(os.path.abspath(__file__)))}
    return None


def workload_config(args, world):
    return {"workload": f"{args.variant} loss+grad step, global B={args.batch}, d={args.dim}, "
                        f"N={args.n_train} u table (BASELINE.json metric config)",
            "variant": args.variant, "global_batch": args.batch, "local_batch": args.batch // world,
            "dim": args.dim, "n_train": args.n_train, "world": world,
            "parallelism": f"dp{world} (anchor slices; NVLink peer all-gathers of E and the scalar payload)" if world > 1
                           else "dp1",
            "l2": "flushed between timed steps (256 MiB memset)", "tables": "warm u (log10 u ~ U[-8,0])",
            **({"tau_init": args.tau} if getattr(args, "tau", None) is not None else {})}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="fastclip_v3")
    ap.add_argument("--batch", type=int, default=5120)
    ap.add_argument("--dim", type=int, default=512)
    ap.add_argument("--n-train", type=int, default=2_700_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tau", type=float, default=None, help="temperature.init (default: the variant's)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as tdist
    import paper_2407_01445_b200 as P
    from paper_2407_01445_b200 import synthetic as S

    world, rank, local = dist_env()
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    # rank 0's stdout carries exactly one JSON line: libraries that print to fd 1 (NCCL's version
    # banner, warnings) are redirected to stderr, the line goes to a duplicate of the real stdout
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)
    B, d, N = args.batch, args.dim, args.n_train
    if B % world:
        raise SystemExit("global batch must be divisible by the number of GPUs")
    Bl = B // world

    cfg = P.config_defaults(args.variant, N, dim=d, local_batch=Bl, world=world, rank=rank, device=local)
    if args.tau is not None:
        cfg.tau_init = args.tau
    if world > 1:
        obj = [P.nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0)
        for i, b in enumerate(obj[0]):
            cfg.nccl_id[i] = b
    step = P.LossStep(cfg)
    step.load_tables(u1=S.warm_u(N, 1), u2=S.warm_u(N, 2))

    n_sets = 4
    host_sets = make_inputs(B, d, N, world, rank, n_sets)
    dev_sets = [(torch.from_numpy(a.view(np.int16)).to(dev).view(torch.bfloat16),
                 torch.from_numpy(b.view(np.int16)).to(dev).view(torch.bfloat16),
                 torch.from_numpy(i).to(dev)) for a, b, i in host_sets]
    de1 = torch.empty(Bl, d, device=dev, dtype=torch.float32)
    de2 = torch.empty(Bl, d, device=dev, dtype=torch.float32)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    gamma = 0.6   # cosine inner LR at epoch 9 of 18 with gamma_min 0.2 (SPEC anchor)
    eps = 1e-14

    def barrier():
        if world > 1:
            tdist.barrier()

    def note(msg):
        if os.environ.get("FC_BENCH_TRACE"):
            print(f"[bench rank {rank}] {msg}", file=sys.stderr, flush=True)

    note("init done")
    # input set j % n_sets at the step's global index j everywhere: with K > 1 the step graphs are
    # keyed by (input set, step parity), and this pairing repeats every n_sets steps, so warm-up
    # steps covering n_sets consecutive indices capture every graph the timed steps replay (no
    # capture inside the timed region)
    args.warmup = max(args.warmup, n_sets)
    for i in range(args.warmup):
        e1, e2, ids = dev_sets[i % n_sets]
        step.step(e1, e2, ids, gamma, eps, de1, de2, stream)
    torch.cuda.synchronize()
    sc = step.scalars()
    note("warmup done")

    # ---------------- device-timed steps (CUDA-graph replay, no host sync inside) ----------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        flush.zero_()
        e1, e2, ids = dev_sets[(args.warmup + i) % n_sets]
        starts[i].record(stream)
        step.step(e1, e2, ids, gamma, eps, de1, de2, stream)
        ends[i].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    sc = step.scalars()
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    note("per-step us: " + " ".join(f"{1e3 * x:.0f}" for x in ms))
    total_ms = float(sum(ms))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = 1e3 / ms_per_step
    note("timed steps done")

    # ---------------- per-kernel durations: CUDA events between the step's phases ----------------
    # (event-record nodes inside the replayed graph, same stream, same inputs; K more steps)
    step.enable_phase_timing(args.steps)
    for i in range(2):
        e1, e2, ids = dev_sets[i % n_sets]
        step.step(e1, e2, ids, gamma, eps, de1, de2, stream)
    torch.cuda.synchronize()
    step.enable_phase_timing(args.steps)   # fresh event ring: slot i <-> timed step i
    for i in range(args.steps):
        flush.zero_()
        e1, e2, ids = dev_sets[i % n_sets]
        step.step(e1, e2, ids, gamma, eps, de1, de2, stream)
    torch.cuda.synchronize()
    # per-phase median over the timed steps (robust to a single late event record)
    phase_runs = {k: [] for k in P.fastclip.PHASES}
    for i in range(args.steps):
        for k, v in step.phase_times(i).items():
            phase_runs[k].append(v)
    phases = {k: (statistics.median(v) if v else 0.0) for k, v in phase_runs.items()}
    step.disable_phase_timing()
    note("phase timing done")

    # ---------------- end to end through the public API (host buffers) ----------------
    e2e = None
    if not args.no_e2e:
        # one pinned host record per input set: [E1 | E2 | ids] bytes (one H2D copy per step), and
        # one pinned [dE1 | dE2] record per output buffer (one D2H copy per step)
        ne = Bl * d * 2
        h2d = 2 * ne + Bl * 4
        rec = []
        for a, b, i in host_sets:
            r = torch.empty(h2d, dtype=torch.uint8).pin_memory()
            r[:ne].copy_(torch.from_numpy(a.view(np.uint8).reshape(-1)))
            r[ne:2 * ne].copy_(torch.from_numpy(b.view(np.uint8).reshape(-1)))
            r[2 * ne:].copy_(torch.from_numpy(i.view(np.uint8)))
            rec.append(r)
        staging = [torch.empty(h2d, dtype=torch.uint8, device=dev) for _ in range(2)]
        views = [(st_[:ne].view(torch.bfloat16).view(Bl, d), st_[ne:2 * ne].view(torch.bfloat16).view(Bl, d),
                  st_[2 * ne:].view(torch.int32)) for st_ in staging]
        outs = [torch.empty(2, Bl, d, device=dev, dtype=torch.float32) for _ in range(2)]
        host_out = [torch.empty(2, Bl, d, dtype=torch.float32).pin_memory() for _ in range(2)]
        d2h = 2 * Bl * d * 4 + 48   # dE1, dE2 (fp32) + the step scalars
        # pipelined feed through the public API: an upload stream copies step i+1's record (pinned
        # -> double-buffered device staging) while step i computes, and a download stream reads
        # step i-1's dE1 / dE2 back (double-buffered outputs -> pinned host); the two copy streams
        # use PCIe's two directions at once. Every step pays its own H2D copy of E1 / E2 / ids and
        # the D2H read of its gradients and scalars (loss / G_tau / tau, mapped pinned memory).
        up = torch.cuda.Stream(dev)
        down = torch.cuda.Stream(dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        computed = [torch.cuda.Event() for _ in range(2)]
        drained = [torch.cuda.Event() for _ in range(2)]
        for ev in consumed + drained:
            ev.record(stream)
        for i in range(4):   # warm the staging / output graphs (an even count: buffer i % 2 meets the same step parity below)
            staging[i % 2].copy_(rec[i % n_sets])
            v = views[i % 2]
            step.step(v[0], v[1], v[2], gamma, eps, outs[i % 2][0], outs[i % 2][1], stream)
        barrier()
        torch.cuda.synchronize()
        e_start = torch.cuda.Event(enable_timing=True)
        e_end = torch.cuda.Event(enable_timing=True)
        e_start.record(stream)
        up.wait_event(e_start)
        down.wait_event(e_start)
        for i in range(args.steps):
            b = i % 2
            with torch.cuda.stream(up):
                up.wait_event(consumed[b])          # step i-2 finished reading this buffer
                staging[b].copy_(rec[i % n_sets], non_blocking=True)
                copied[b].record(up)
            stream.wait_event(copied[b])
            stream.wait_event(drained[b])           # step i-2's gradients are on the host
            v = views[b]
            step.step(v[0], v[1], v[2], gamma, eps, outs[b][0], outs[b][1], stream)
            consumed[b].record(stream)
            computed[b].record(stream)
            with torch.cuda.stream(down):
                down.wait_event(computed[b])
                host_out[b].copy_(outs[b], non_blocking=True)
                drained[b].record(down)
        stream.wait_stream(down)
        e_end.record(stream)
        _ = step.scalars()
        torch.cuda.synchronize()
        tot = e_start.elapsed_time(e_end)
        if world > 1:
            t = torch.tensor([tot], device=dev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            tot = float(t.item())
        e2e = {"value": 1e3 * args.steps / tot, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": tot / args.steps}

    if rank != 0:
        if world > 1:
            tdist.barrier()
            tdist.destroy_process_group()
        return 0

    # ---------------- roofline ----------------
    peak, peak_sus, hbm, peak_kind = peaks()
    Bd = float(B) * float(Bl) * float(d)
    # SURVEY.md §8d algorithmic flops: K=1: 6 B^2 d (S once + two weight GEMMs);
    # K>1: 8 Bl B d per rank (row block + column block + two GEMMs).
    step_flops = 6.0 * B * B * d if world == 1 else 8.0 * Bd
    # the step's algorithmic flops split over the three tensor kernels (shares sum to F):
    # S (2 B^2 d at K=1, 4 Bl B d at K>1) is credited half to each similarity pass.
    s_share = (1.0 * B * B * d) if world == 1 else 2.0 * Bd
    per_kernel_flops = {"pass1_stats": s_share, "pass2_q": s_share, "grad_gemm": 4.0 * Bd}
    # executed: the K = 1 pass 1 multiplies S once (row and column statistics from one tile), K > 1
    # runs both segments; pass 2 recomputes S (K = 1: once, Q^T shared) / both segments
    exec_flops = {"pass1_stats": (2.0 if world == 1 else 4.0) * Bd, "pass2_q": (2.0 if world == 1 else 4.0) * Bd,
                  "grad_gemm": 4.0 * Bd}
    tensor_phases = ["pass1_stats", "pass2_q", "grad_gemm"]
    dom = max(tensor_phases, key=lambda k: phases[k])
    t_dom = phases[dom] * 1e-3
    ach = per_kernel_flops[dom] / t_dom / 1e12 if t_dom > 0 else 0.0
    roofline = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "traffic": (ncu_traffic(dom) or {}).get("bytes"),
                "traffic_source": ncu_traffic(dom), "peak_kind": f"{peak_kind} bf16 burst",
                "executed_tflops": exec_flops[dom] / t_dom / 1e12 if t_dom > 0 else 0.0,
                "algorithmic_flops_per_launch": per_kernel_flops[dom]}
    # the table kernel (K2: fc_anchor_kernel, the "tables_tau" phase): SURVEY.md §8(d) algorithmic
    # bytes per id -- 4 B id + 16 B u read + 16 B u write, +128 B for the v2 tau / Adam state --
    # over its measured duration, against the HBM peak; it is latency-bound (one dependent fp64
    # chain per anchor), which the fraction makes explicit
    indiv = args.variant in ("fastclip_v2", "isogclr")
    k2_bytes = float(Bl) * (36.0 + (128.0 if indiv else 0.0))
    t_k2 = phases.get("tables_tau", 0.0) * 1e-3
    k2 = {"kernel": "fc_anchor_kernel", "bound": "hbm", "algorithmic_bytes": k2_bytes,
          "achieved": k2_bytes / t_k2 / 1e9 if t_k2 > 0 else 0.0, "peak": hbm, "unit": "GB/s",
          "frac": (k2_bytes / t_k2 / 1e9) / hbm if t_k2 > 0 else 0.0,
          "traffic": (ncu_traffic("tables_tau") or {}).get("bytes"),
          "note": "latency-bound: one fp64 dependent chain per anchor (partials -> g -> EMA -> weights -> logs)"}
    step_ach = step_flops / (ms_per_step * 1e-3) / 1e12
    step_roofline = {"achieved": step_ach, "peak": peak, "unit": "TFLOP/s", "frac": step_ach / peak,
                     "frac_of_sustained": step_ach / peak_sus, "algorithmic_flops_per_step": step_flops}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference_step(B, d, N, args.variant, lambda m: print(m, file=sys.stderr))
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as ex:  # the checker is absent on this box
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {ex}"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": workload_config(args, world), "e2e": e2e,
            "gpu_launches": step.kernels_per_step * args.steps,
            "roofline": roofline, "step_roofline": step_roofline, "table_kernel": k2,
            "phases_ms": phases, "clocks": clk, "cpu_baseline": cpu,
            "last_step": {"loss": sc.loss, "gtau": sc.gtau, "tau": sc.tau, "exp_clamps": sc.exp_clamps}}
    print(json.dumps(line), file=out, flush=True)
    if world > 1:   # torch's process group first, then the loss step's own communicator
        tdist.barrier()
        tdist.destroy_process_group()
        note("process group destroyed")
    step.close()
    note("loss step closed")
    return 0


if __name__ == "__main__":
    sys.exit(main())
