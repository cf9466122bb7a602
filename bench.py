#!/usr/bin/env python
"""bench.py -- batched subsequence DTW (arXiv 2403.06931) on B200.

Metric (BASELINE.json): GCUPS = cell updates / s = Z*N*M / t, whole job over all
ranks.  One "step" = one pass of the whole hot path over one batch: query
z-normalisation + wavefront DP + min/argmin epilogue (+ the one all-gather of
per-query records when N>1), through the public API (sdtw_batch) on inputs
already resident in HBM.  Default workload (`--config c3`): 512 x 2,000-sample
queries against a 10M-sample synthetic nanopore-like reference (BASELINE config 3),
STRONG scaling: at N GPUs each rank takes 512/N queries (64 at N=8), the metric's
"512x2000 queries, 1/2/4/8 B200".  `--scaling weak` keeps 512 queries per GPU
(4,096 at 8 GPUs = config 4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c4|c5_500|...]
                    [--impl ours|reference] [--scaling weak|strong]

Timing: per step, L2 is flushed (a 256 MiB write, outside the timed window), then
CUDA events on torch's current stream bracket the step; barrier + synchronize on
both sides; rank 0 reports the max over ranks.  The DP kernel is also timed on
its own stream by the library (SDTW_OPT_PROFILE) for the roofline object.
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the
same workload on the host cores (rank 0 only).
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

# ALU roofline: SMs x 128 FP32 lanes x f_SM / (SASS issue slots per cell)
LANES_PER_SM = 128
# Register-file bound: per SMSP every instruction holds the operand-read stage
# for max(#distinct even-bank, #distinct odd-bank) registers (B300_MICROARCH.md "RF banking"),
# whatever pipe it issues to.  Lower bound of those cycles per warp-instruction group and the
# cells that group computes per lane, for each cell mix:
#   packed fp32: FADD2 (x,y pairs: 2) + FFMA2 (t,m pairs: 2) + 2 FMNMX3 (3 scalars: 2 each) = 8 / 2 cells
#   half2: VHMNMX (2) + HADD2 (1) + HFMA2 (1) = 4 / 2 cells
#   scalar fp32 / uint8: FMNMX3|VIMNMX3 (2) + FADD|IADD (1) + FFMA|IMAD (1) = 4 / 1 cell
#   uint8 pruned: + IMAD t^2 (1) + ISETP (1) + IADD d+m (1) + SEL (1) - (t*t+m fused) = 7 / 1 cell
#   start index (forward): + 2 FSETP (1 each) + 2 SEL (1 each) = 8 / 1 cell
RF_CYCLES_PER_CELL = {"q8": 4.0, "q8_prune": 7.0, "half2": 2.0, "packed_fma": 4.0, "scalar_fma": 4.0,
                      "packed_fma_trace": 8.0, "scalar_fma_trace": 8.0}
SASS_PER_CELL = {"q8": 3.0, "q8_prune": 6.0, "half2": 1.5, "packed_fma": 2.0, "scalar_fma": 3.0, "scalar_nofma": 4.0, "packed_nofma": 3.5,
                 "packed_fma_trace": 6.0, "scalar_fma_trace": 7.0}


def gsps(floats: float, ms: float) -> float:
    """PAPER.md Eq. 3: floatsProcessed / (milliseconds * 1e9 / 1000)."""
    if ms <= 0:
        raise ValueError("ms must be > 0")
    return floats / (ms * 1e9 / 1000.0)


def _traffic(config, w, precision=32):
    """DRAM bytes (read + write) per DP launch from the committed ncu capture of this
    workload (profiles/traffic_<config>.json, written by scripts/ncu_traffic.py from
    `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum`), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_%s.json" % config)) as f:
            t = json.load(f)
        if (int(t["Z"]) == int(w["Z_local"]) and int(t["N"]) == w["N"] and int(t["M"]) == w["M"]
                and int(t.get("precision", 32)) == precision):
            return float(t["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


def _issue_counts(config, w, precision=32):
    """Measured instruction counts per cell of the DP kernel from the committed ncu capture of
    this workload (profiles/issue_<config>.json, written by scripts/ncu_issue.py from
    `ncu --set full` of one DP launch): issue slots per cell = warp instructions x 32 / cells,
    thread instructions per cell, issue-active fraction.  None when no capture matches."""
    try:
        with open(os.path.join(ROOT, "profiles", "issue_%s.json" % config)) as f:
            t = json.load(f)
        if (int(t["Z"]) == int(w["Z_local"]) and int(t["N"]) == w["N"] and int(t["M"]) == w["M"]
                and int(t.get("precision", 32)) == precision):
            return {"issue_slots_per_cell_ncu": t["issue_slots_per_cell"],
                    "thread_inst_per_cell_ncu": t["thread_inst_per_cell"],
                    "issue_active_ncu": t["issue_active"], "ncu_capture": t["source"]}
    except Exception:
        pass
    return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                row = [x.strip() for x in out.split(",")] if out else []
                if len(row) >= 8:                   # skip error text / partial rows
                    self.samples.append(row)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for n, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "power_w_max": max(pw) if pw else None,
                "samples": len(self.samples)}


def _workload(cfg_name: str, rank: int, world: int, scaling: str):
    from datagen import CONFIGS, nanopore_queries, nanopore_reference
    cfg = dict(CONFIGS[cfg_name])
    Z, N, M, seed = cfg["Z"], cfg["N"], cfg["M"], cfg["seed"]
    if scaling == "weak":
        Zl, first = Z, rank * Z
        Zg = Z * world
    else:
        per = -(-Z // world)
        first = rank * per
        Zl = max(0, min(Z, first + per) - first)
        Zg = Z
    if cfg.get("cbf"):
        from datagen import cbf_batch, cbf_reference
        Q = cbf_batch(Zl, N, seed + 1000 * first)
        return Q, cbf_reference(M, seed), dict(Z=Zg, Z_local=Zl, N=N, M=M, seed=seed, start=cfg["start"])
    Y = nanopore_reference(M, seed)
    if cfg.get("ragged"):
        from datagen import nanopore_ragged
        Q, off = nanopore_ragged(Zl, M, seed, *cfg["ragged"], first_query=first)
        return Q, Y, dict(Z=Zg, Z_local=Zl, N=N, M=M, seed=seed, start=cfg["start"], offsets=off,
                          cells_local=float(off[-1]) * M)
    Q = nanopore_queries(Zl, N, M, seed, first_query=first)
    if cfg.get("straddle"):
        # every `every`-th query matches a `stride`x oversampled reference region placed 1,000
        # columns before a boundary of the 6-segment speculative plan (OPT_SEGMENTS=6 is set
        # for this config; boundary s = floor(s*Pr/6) rounds x columns per round), so its path
        # runs N*stride - 1,000 columns past the boundary -- beyond the correction pass (2
        # rounds = 7,680 columns at N = 2,000)
        import paper_2403_06931_b200 as sd
        from datagen import straddle_workload
        every, stride = cfg["straddle"]
        cols = sd.round_columns(N)
        Pr = -(-M // cols)
        bounds = [((s * Pr) // 6) * cols for s in range(1, 6)]
        ks = [k for k in range(Zl) if (first + k) % every == 0]
        per = -(-len(ks) // len(bounds))
        Y, Qs = straddle_workload(Y, bounds, per, N, stride, 1000, seed)
        Q[ks] = Qs[:len(ks)]
    return Q, Y, dict(Z=Zg, Z_local=Zl, N=N, M=M, seed=seed, start=cfg["start"])


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on a bounded sample, host cores."""
    import oracle
    from datagen import CONFIGS, nanopore_queries, nanopore_reference
    cfg = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    N = cfg["N"]
    # bounded sample: `threads` queries x N against the first Ms reference samples,
    # sized for ~2-4 s per step at ~0.3 GCUPS per core
    Ms = int(min(cfg["M"], max(2000, 1.0e9 / N)))
    if cfg.get("cbf"):
        from datagen import cbf_batch, cbf_reference
        Y = cbf_reference(cfg["M"], cfg["seed"])[:Ms]
        Q = cbf_batch(threads, N, cfg["seed"])
    else:
        Y = nanopore_reference(cfg["M"], cfg["seed"])[:Ms]
        Q = nanopore_queries(threads, N, cfg["M"], cfg["seed"])
    Yn = oracle.znorm(Y[None])[0]
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        Qn = oracle.znorm(Q)
        oracle.sdtw(Qn, Yn, fma=True, start=cfg["start"], threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    cells = float(threads) * N * Ms
    tot = sum(times)
    val = cells * len(times) / tot / 1e9
    sample = "%d queries x %d samples (config %s inputs) vs the first %d reference samples, %d host threads" % (
        threads, N, args.config, Ms, threads)
    line = {
        "impl": "reference", "metric": "GCUPS", "value": val, "unit": "GCUPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic nanopore-like (datagen), seeded",
        "config": {"workload": args.config, "sample": sample},
        "cpu_baseline": {"value": val, "unit": "GCUPS", "cores": threads, "kind": "oracle", "sample": sample,
                         "host": host_cpu()},
        "e2e": {"value": val, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def host_cpu():
    """lscpu model name, sockets, physical cores and hardware threads of this host."""
    info = {"model": None, "sockets": None, "cores": None, "threads": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        soc = int(kv.get("Socket(s)", "0") or 0)
        cps = int(kv.get("Core(s) per socket", "0") or 0)
        info["sockets"] = soc or None
        info["cores"] = soc * cps or None
        info["threads"] = int(kv.get("CPU(s)", info["threads"]) or info["threads"])
    except Exception:
        pass
    return info


def cpu_baseline_leg(args, Q, Y, N):
    """The oracle timed on the host cores, rank 0, N=1, bounded sample (~10-30 s)."""
    import oracle
    threads = os.cpu_count() or 1
    Ms = int(min(Y.shape[0], max(2000, 2.0e9 / N)))
    if Q.ndim == 1:   # ragged batch: time the oracle on a slab of the same samples cut at length N
        Q = Q[:(Q.shape[0] // N) * N].reshape(-1, N)
    nq = min(Q.shape[0], threads)
    Yn = oracle.znorm(Y[:Ms][None])[0]
    Qn = oracle.znorm(Q[:nq])
    t0 = time.perf_counter()
    oracle.sdtw(Qn, Yn, fma=True, threads=threads)
    dt = time.perf_counter() - t0
    cells = float(nq) * N * Ms
    return {"value": cells / dt / 1e9, "unit": "GCUPS", "cores": threads, "kind": "oracle",
            "sample": "%d queries x %d vs first %d reference samples of the same inputs, %d threads, %.1f s"
                      % (nq, N, Ms, threads, dt), "host": host_cpu()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--half", action="store_true",
                    help="packed-half precision (SDTW_OPT_PRECISION=16, SURVEY NEXT-1: the paper's __half2)")
    ap.add_argument("--q8", action="store_true",
                    help="uint8 codebook (sdtw_batch_q8, SURVEY NEXT-3, PAPER.md P:L165): integer cells")
    ap.add_argument("--q8-prune", type=int, default=-1,
                    help="with --q8: INF-prune cells whose codes differ by more than TAU (-1: off)")
    ap.add_argument("--path", action="store_true",
                    help="step = sdtw_path (start index + full warp path, SURVEY NEXT-2)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 collective backend; gloo lets several ranks share one GPU (a functional "
                         "check of the multi-rank path on a one-GPU box -- not a scaling number)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return

    import torch
    import torch.distributed as dist
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    comm = None
    tdev = dev                       # where the max-over-ranks reductions run
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
            tdev = torch.device("cpu")
        comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size(), "rank": rank,
                "nccl_version": ".".join(str(v) for v in torch.cuda.nccl.version()),
                "ranks_per_gpu": max(1, -(-world // ndev))}
        print("[bench] communicator: %s world_size=%d rank=%d local_rank=%d device=%s nccl=%s"
              % (comm["backend"], comm["world_size"], rank, local, dev, comm["nccl_version"]),
              file=sys.stderr, flush=True)

    import paper_2403_06931_b200 as sd
    from paper_2403_06931_b200.distributed import distributed_batch
    if args.half:
        sd.set_option(sd.OPT_PRECISION, 16)
    if args.q8:
        sd.set_option(sd.OPT_Q8_PRUNE, args.q8_prune)

    if args.config == "c3_straddle":
        sd.set_option(sd.OPT_SEGMENTS, 6)
    Q, Y, w = _workload(args.config, rank, world, args.scaling)
    N, M = w["N"], w["M"]
    trace = bool(w["start"])
    sd.set_reference(torch.from_numpy(Y).to(dev))
    Qd = torch.from_numpy(Q).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    trace = trace or args.path

    ragged = "offsets" in w
    if ragged:
        if world > 1 or args.path:
            raise SystemExit("ragged configs run on one GPU without --path")
        off_d = torch.from_numpy(w["offsets"]).to(dev)

    def step():
        if ragged:
            return sd.batch_ragged(Qd, off_d)
        if world > 1:
            return distributed_batch(Qd, traceback=trace, pre_sharded=True, device=dev, path=args.path)
        if args.path:
            return sd.path(Qd)
        if args.q8:
            return sd.batch_q8(Qd)
        return sd.traceback(Qd) if trace else sd.batch(Qd)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    dp_ms = []
    recomputed = 0
    launches0 = sd.launch_count()
    # nvidia-smi -i takes the physical index or the UUID; the UUID survives CUDA_VISIBLE_DEVICES
    # remapping and several ranks sharing one GPU
    try:
        smi_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        smi_id = str(dev.index)
    sampler = ClockSampler(smi_id)
    with sd.options(OPT_PROFILE=1), sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            dp_ms.append(sd.profile()[0])
            recomputed += sd.spec_recomputed()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = sd.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    cells_step = w["cells_local"] * world if ragged else float(w["Z"]) * N * M
    value = cells_step * args.steps / (tot_ms / 1e3) / 1e9

    # roofline of the dominant kernel (the DP kernel), measured on its own stream
    peaks, src = _peaks()
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    popt = sd.get_option(sd.OPT_PACKED)
    # the library's auto choice (sdtw_api.cu plan): packed chains for cost/end and for the
    # checkpointed start index (OPT_START 0/2: the cost/end kernel + window walk-back)
    ckpt_start = trace and sd.get_option(sd.OPT_START) != 1 and popt in (-1, 1)
    packed = popt > 0 or (popt < 0 and (not trace or ckpt_start))
    mix = "half2" if args.half else ("packed" if packed else "scalar") + "_fma" + (
        "_trace" if trace and not ckpt_start else "")
    if args.q8:
        mix = "q8_prune" if 0 <= args.q8_prune < 255 else "q8"
    k = SASS_PER_CELL[mix]
    peak = sms * LANES_PER_SM * fmax * 1e6 / k / 1e9
    peak3 = sms * LANES_PER_SM * fmax * 1e6 / 3.0 / 1e9
    dp_avg = statistics.mean(dp_ms)
    achieved = (w["cells_local"] if ragged else float(w["Z_local"]) * N * M) / (dp_avg / 1e3) / 1e9
    clocks = sampler.summary()
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "GCUPS", "frac": achieved / peak,
            "traffic": _traffic(args.config, w, 16 if args.half else (8 if args.q8 else 32)), "sass_per_cell": k, "peak_source": "%s sm_max_mhz=%.0f x %d SMs x %d lanes / %g"
            % (src, fmax, sms, LANES_PER_SM, k),
            "headline_peak_k3": peak3, "headline_frac_k3": achieved / peak3,
            "dp_kernel_ms": dp_avg}
    if clocks.get("sm_mhz"):
        roof["frac_at_sampled_clock"] = achieved / (peak * clocks["sm_mhz"] / fmax)
    if mix in RF_CYCLES_PER_CELL:
        # 4 SMSPs x 32 lanes per SM: cells / SM / cycle = 128 / RF cycles per cell
        rf_peak = sms * 4 * 32 / RF_CYCLES_PER_CELL[mix] * fmax * 1e6 / 1e9
        roof["rf_bound"] = {"peak": rf_peak, "frac": achieved / rf_peak,
                            "smsp_rf_cycles_per_warp_cell": RF_CYCLES_PER_CELL[mix],
                            "model": "operand reads: max(#even, #odd) distinct registers per instruction "
                                     "per SMSP (B300_MICROARCH.md RF banking); DESIGN.md §5"}
    if not args.half and not args.q8:
        # the min alone: FMNMX3 with nothing else in the loop issues 47.5 cells per SM-cycle at 16
        # warps/SM (profiles/r02p_mixbench.txt, "FMNMX3 only"): any one-FMNMX3-per-cell fp32
        # formulation is capped there before a single add
        fm_peak = sms * 47.5 * fmax * 1e6 / 1e9
        roof["fmnmx3_ceiling"] = {"peak": fm_peak, "frac": achieved / fm_peak,
                                  "source": "measured FMNMX3-only loop, 47.5 cells/SM/cycle (profiles/r02p_mixbench.txt)"}
    meas = _issue_counts(args.config, w, 16 if args.half else (8 if args.q8 else 32))
    if meas:
        roof.update(meas)
    if ckpt_start:
        roof["start_index"] = ("checkpointed (DESIGN.md §15): cost/end DP kernel with round checkpoints, "
                               "then window DP + walk-back; DP kernel %.1f ms of a %.1f ms step"
                               % (dp_avg, tot_ms / args.steps))
    elif trace:
        # the start-index cell needs 5 ALU-pipe ops (FMNMX3 + 2 FSETP + 2 SEL; the ALU pipe
        # issues 16 lanes/clk/SMSP): that pipe, not issue, binds it (ncu: alu 72 % busy)
        alu_peak = sms * 64 * fmax * 1e6 / 5.0 / 1e9
        roof["alu_pipe_peak"] = alu_peak
        roof["alu_pipe_frac"] = achieved / alu_peak

    # e2e: the same metric through the public API with host buffers (pinned), copies inside
    e2e = None
    if not args.no_e2e:
        Qh = torch.from_numpy(Q).pin_memory()
        api = sd.path if args.path else (sd.traceback if trace else (sd.batch_q8 if args.q8 else sd.batch))
        if ragged:
            api = lambda q: sd.batch_ragged(q, w["offsets"])  # noqa: E731
        api(Qh.numpy())
        ts = []
        for i in range(max(1, min(args.steps, 3))):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            # device-timed like the main number: the library enqueues the pinned-host
            # H2D copy, the kernels and the D2H result copy on this stream
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if world > 1:   # the gathered records stay on the GPU: read the costs back to the host
                distributed_batch(Qh.numpy(), traceback=trace, pre_sharded=True, device=dev, path=args.path)[0].cpu()
            else:
                api(Qh.numpy())
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        te = sum(ts)
        if world > 1:
            t = torch.tensor([te], dtype=torch.float64, device=tdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": cells_step * len(ts) / te / 1e9, "unit": "GCUPS",
               "h2d_bytes_per_step": int(Q.nbytes) * world,
               "d2h_bytes_per_step": int(w["Z"]) * (4 + 8 + (8 if trace else 0) + (8 * N if args.path else 0))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(args, Q, Y, N)

    if rank == 0:
        line = {
            "metric": "GCUPS", "value": value, "unit": "GCUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f16" if args.half else ("i32 (u8 codes)" if args.q8 else "f32"),
            "data": "synthetic nanopore-like signals (datagen, seeded); random reference, no trained weights",
            "config": {"workload": "%s: %d x %d queries vs %d-sample reference%s" % (
                args.config, w["Z"], N, M, " (start index on)" if trace else ""),
                "queries_per_gpu": w["Z_local"], "N": N, "M": M, "normalize": True, "fma": True,
                "packed": packed, "l2": "flushed (256 MiB write) before every timed step",
                "parallelism": "query-sharded x%d (%s scaling), reference replicated, one all-gather of "
                               "per-query records" % (world, args.scaling),
                "schedule": {0: "auto (speculative round-segments with exact correction, DESIGN.md §13)",
                             1: "one CTA per ring", 2: "sequential round-segments",
                             3: "speculative round-segments"}[sd.get_option(sd.OPT_SCHED)]},
            "gpu_launches": launches, "roofline": roof, "clocks": clocks,
            "spec_recomputed": recomputed, "build": sd.build_info(), "comm": comm,
            "gsps_eq3": gsps(float(w["Z"]) * N, tot_ms / args.steps),
            "e2e": e2e, "cpu_baseline": cpu,
        }
        if args.q8:
            # accuracy metric of the approximation: end index of the uint8 path
            # against the fp32 path (bit-exact with the fp32 oracle) on this batch, untimed
            cq, eq = step()
            ef = sd.batch(Qd)[1]
            d = (eq.to(torch.int64) - ef).abs()
            line["q8"] = {"prune_tau": args.q8_prune, "codebook": [float(v) for v in sd.q8_codebook()],
                          "end_exact_vs_fp32": float((d == 0).double().mean().item()),
                          "end_within_8_vs_fp32": float((d <= 8).double().mean().item()),
                          "all_paths_pruned": int((cq >= (1 << 30)).sum().item())}
            line["config"]["workload"] += " (uint8 codebook%s)" % (
                ", INF pruning tau=%d" % args.q8_prune if 0 <= args.q8_prune < 255 else "")
        if args.path:
            import torch as _t
            c, e, st, lo, hi = [_t.as_tensor(np.asarray(a.cpu() if hasattr(a, "cpu") else a)) for a in step()]
            L = (e - st + 1).double()
            line["path"] = {"window_cells_per_step": float((L * N).sum().item()),
                            "path_cells_per_step": float((hi.double() - lo.double() + 1).sum().item()),
                            "step_ms_incl_path": tot_ms / args.steps, "dp_kernel_ms": dp_avg,
                            "non_dp_share": 1.0 - dp_avg / (tot_ms / args.steps)}
            line["config"]["workload"] += " + full warp path (sdtw_path)"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
