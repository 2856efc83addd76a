"""Benchmark: N-1-evaluated topologies/s of the device-resident MapElites loop.

Workload (default, BASELINE.json configs[3], the largest single-GPU config):
synthetic TSO-scale 7k-bus / 10.5k-branch grid with 500 splittable stations,
a 16384-candidate batch per generation, full single-branch N-1 over every
listed contingency, 1 timestep. One step = one MapElites generation: device
mutation/crossover of every lane, DC N-1 evaluation of every lane, archive
insert (qd_optimizer.cpp:376-401), launched as one CUDA graph. --config
cfg1|cfg2|cfg3 select the other BASELINE configs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4|cfg3|cfg2|cfg1] [--impl b200|reference]

Multi-GPU (torchrun): one island per rank (own seed, own archive), archives
merged every --merge-every generations (NCCL allgather of the archive blobs +
device merge kernel, islands.py), weak scaling, device time = max over ranks. --impl reference times the reference's
CPU algorithm (the oracle restatement, oracle/, threaded like
dc_engine.cpp:446-465) on this host on the same workload.
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

L2_BYTES = 126 * 2 ** 20

CONFIGS = {
    "cfg1": dict(workload="grid14_congested (bundled), batch 64, full N-1, 1 busbar outage", batch=64),
    "cfg2": dict(workload="synthetic 1k-bus/1.5k-branch grid, 4096-candidate batch, full N-1, 1 timestep",
                 batch=4096),
    "cfg3": dict(workload="synthetic 2k-bus grid, bus splitting on 100 substations, 24 timesteps, N-1 over all "
                          "non-reserved branches", batch=4096),
    "cfg4": dict(workload="synthetic TSO-scale 7k-bus/10.5k-branch grid, 500 splittable stations, "
                          "16384-candidate batch, full N-1", batch=16384),
}


def grid_text(cfg: str) -> str:
    if cfg == "cfg1":
        return open(os.path.join(ROOT, "tests", "golden", "data", "grid14_congested.json")).read()
    from tools.synth_grid import config_json
    return config_json(cfg)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # NCCL over NVLink/NVSwitch; TGB_DIST_BACKEND=gloo (host-staged exchange,
        # ranks may share a GPU) is the single-GPU test harness of the N>1 path
        dist.init_process_group(os.environ.get("TGB_DIST_BACKEND", "nccl"))
    return world, rank, local


def max_over_ranks(x: float, world: int, dev: int) -> float:
    """Max of a per-rank time over all ranks (device tensor for NCCL, host for gloo)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}" if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # the timed region can be shorter than nvidia-smi's start-up: wait for
            # its first sample so the region is covered
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def mark(self):
        """Start of the timed region: samples from here on describe it."""
        self.start = len(self.lines)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        start = getattr(self, "start", 0)
        lines = self.lines[start:] if len(self.lines) > start else self.lines[-1:]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def _reference_loop(text: str, gens_warm: int, gens_timed: int, gen_seconds: float, batch_cap: int):
    """The reference's own MapElites loop (run_optimizer, qd_optimizer.cpp:344-417,
    restated in oracle/) on this host: mutate / crossover from its archive,
    DcContext::evaluate_batch on all host threads (dc_engine.cpp:446-465),
    Repertoire::insert. The per-generation batch is a bounded sample of the
    workload's batch, sized from a probe so one generation takes about
    gen_seconds. Returns (topologies/s over the timed generations, lanes per
    generation, timed seconds, cores)."""
    from oracle.oracle import OracleContext, qd_config
    orc = OracleContext(text)
    cores = os.cpu_count() or 1
    probe = orc.random_genomes(max(16, cores), 3, 2, seed=11)
    t = orc.time_evaluate_batch(probe, 3, 2, 1) / len(probe)  # seconds per lane, threaded
    lanes = int(max(16, min(batch_cap, gen_seconds / max(t, 1e-9))))
    lanes = min(batch_cap, -(-lanes // cores) * cores)  # whole rounds of the thread fan-out
    gens = gens_warm + gens_timed
    cfg = qd_config(batch_size=lanes, iters_per_epoch=1 << 30, seed=1, max_evaluations=1 + gens * lanes)
    stamps, _ = orc.run_optimizer_timed(cfg)
    assert len(stamps) == gens, (len(stamps), gens)
    dt = float(stamps[-1] - stamps[gens_warm - 1])
    T = n_timesteps(text)  # the reference evaluates one injection vector: one evaluation per timestep
    return lanes * gens_timed / dt / T, lanes, dt * T, cores


def cpu_baseline(text: str, batch_cap: int):
    """cpu_baseline leg (rank 0, N=1): ~10-15 s of the reference loop."""
    value, lanes, dt, cores = _reference_loop(text, 1, 8, 1.5, batch_cap)
    T = n_timesteps(text)
    note = (f"; {T} timesteps = {T} reference evaluations per topology (timed on one profile, rate / {T})"
            if T > 1 else "")
    return {"value": value, "unit": "topologies/s", "cores": cores, "kind": "port",
            "sample": f"the reference's MapElites loop (oracle restatement of run_optimizer): 8 timed generations of "
                      f"{lanes} lanes (bounded sample of the {batch_cap}-lane batch) after 1 warm-up generation, "
                      f"full N-1, evaluate_batch on {cores} threads, {dt:.1f} s{note}"}


def n_timesteps(text: str) -> int:
    return int(json.loads(text).get("timesteps", {}).get("count", 1))


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path on this host (rank 0 only):
    its own MapElites loop, each step one generation of a bounded lane sample."""
    if rank != 0:
        return
    text = grid_text(args.config)
    B = CONFIGS[args.config]["batch"]
    value, lanes, dt, cores = _reference_loop(text, args.warmup, args.steps, 2.0, B)
    T = n_timesteps(text)
    line = {"metric": "N-1-evaluated topologies/sec (DC)", "value": value, "unit": "topologies/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, reference JSON format)",
            "impl": "reference",
            "config": {"workload": CONFIGS[args.config]["workload"], "batch_per_step": lanes,
                       "note": f"each step is one generation of the reference's MapElites loop over a bounded "
                               f"sample of {lanes} lanes (of the {B}-lane batch)"},
            "cpu_baseline": {"value": value, "unit": "topologies/s", "cores": cores, "kind": "port",
                             "sample": f"run_optimizer (oracle restatement): {args.warmup} warm-up + {args.steps} "
                                       f"timed generations of {lanes} lanes, evaluate_batch on {cores} threads"
                                       + (f", x {T} profiles (one reference evaluation per timestep, timed on one)"
                                          if T > 1 else "")},
            "e2e": {"value": value, "unit": "topologies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- AC stage (--stage ac)
AC_CONFIGS = {
    "cfg1": dict(workload="grid14_congested (bundled), 2048 DC-proposed topologies, full AC N-1 validation "
                          "(base case + every contingency)", genomes=2048),
    "ac118": dict(workload="synthetic 118-bus grid with AC data (tools/synth_grid.py with_ac_data), 256 topologies, "
                           "full AC N-1 validation", genomes=256),
}


def ac_grid_text(cfg: str) -> str:
    if cfg == "cfg1":
        return open(os.path.join(ROOT, "tests", "golden", "data", "grid14_congested.json")).read()
    from tools.synth_grid import synth_grid, with_ac_data
    return json.dumps(with_ac_data(synth_grid(118, seed=7, n_stations=6)))


def random_valid_genomes(actions, n: int, n_a: int = 3, n_d: int = 2, seed: int = 5) -> np.ndarray:
    """Valid genomes (distinct stations, distinct disconnections; genome.cpp:41-62)."""
    rng = np.random.default_rng(seed)
    ranges = sorted(actions.station_ranges.items())
    D = len(actions.disconnectables)
    out = np.full((n, n_a + n_d), -1, np.int32)
    for i in range(n):
        ns = int(rng.integers(0, min(n_a, len(ranges)) + 1))
        for j, k in enumerate(rng.choice(len(ranges), ns, replace=False)):
            lo, hi = ranges[k][1]
            out[i, j] = int(rng.integers(lo, hi))
        nd = int(rng.integers(0, min(n_d, D) + 1))
        for j, d in enumerate(rng.choice(D, nd, replace=False)):
            out[i, n_a + j] = int(d)
    return out


def run_ac(args, world, rank):
    """AC validation stage: AcValidator::full_validation for a batch of
    topologies, every (topology, contingency) case solved by the batched device Newton-Raphson.
    One step = one full_validation call through the C ABI with host genomes in and verdicts
    out. --impl reference: the reference algorithm (oracle restatement) on all host cores."""
    cfgname = args.config if args.config in AC_CONFIGS else "cfg1"
    text = ac_grid_text(cfgname)
    n_gen = AC_CONFIGS[cfgname]["genomes"]
    if args.impl == "reference":
        if rank != 0:
            return
        from oracle.oracle import OracleAc, OracleContext
        orc = OracleContext(text)
        oac = OracleAc(orc)
        import paper_2605_10128_b200  # noqa: F401  (not used: genomes below come from numpy)
        K = orc.info["n_contingencies"]
        gen = orc.random_genomes(n_gen, 3, 2, seed=5)
        cores = os.cpu_count() or 1
        cg = np.repeat(np.arange(n_gen), K + 1).astype(np.int32)
        ck = np.tile(np.arange(-1, K, dtype=np.int32), n_gen)
        t0 = time.perf_counter()
        oac.cases(gen, 3, 2, cg[:cores * (K + 1)], ck[:cores * (K + 1)], threads=cores, loading=False)
        per = (time.perf_counter() - t0) / (cores * (K + 1))
        m = int(max(cores * (K + 1), min(len(cg), 2.0 / max(per, 1e-9))))
        times = []
        for _ in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            oac.cases(gen, 3, 2, cg[:m], ck[:m], threads=cores, loading=False)
            times.append(time.perf_counter() - t0)
        dt = sum(times[args.warmup:])
        value = m * args.steps / dt / (K + 1)
        line = {"metric": "AC N-1 validated topologies/sec", "value": value, "unit": "topologies/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1000 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic genomes", "impl": "reference",
                "config": {"workload": AC_CONFIGS[cfgname]["workload"], "cases_per_step": m},
                "cpu_baseline": {"value": value, "unit": "topologies/s", "cores": cores, "kind": "port",
                                 "sample": f"{m} AcNetwork::run_case solves per step (bounded sample) on {cores} "
                                           "threads"},
                "e2e": {"value": value, "unit": "topologies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2605_10128_b200 as P
    from paper_2605_10128_b200.ac import AcContext

    dev = local_device = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    grid = P.grid_from_json_text(text)
    actions = P.build_action_set(grid)
    dc = P.DcContext(grid, actions, P.DcConfig(), device=local_device)
    t_setup = time.perf_counter()
    ac = AcContext(grid, actions, dc, device=dev)
    setup_s = time.perf_counter() - t_setup
    K = grid.n_contingencies
    genomes = random_valid_genomes(actions, n_gen, seed=5 + rank)
    for _ in range(args.warmup):
        ac.full_validation_arrays(genomes, 3, 2)
    l0 = ac.kernel_launches()
    with ClockSampler(dev) as clk:
        clk.mark()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            reason, acc, lo = ac.full_validation_arrays(genomes, 3, 2)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    dt = max_over_ranks(dt, world, dev)
    launches = ac.kernel_launches() - l0
    value = n_gen * args.steps * world / dt
    # iterations per case for the work estimate (one extra probe call)
    cg = np.repeat(np.arange(n_gen), K + 1).astype(np.int32)
    ck = np.tile(np.arange(-1, K, dtype=np.int32), n_gen)
    r = ac.run_cases(genomes, cg, ck, 3, 2, loading=False, voltages=False)
    nb = grid.n_nodes + 3
    nu = 2 * (nb - 1)
    # dense LU (2/3 nu^3) + Jacobian and injections (~ 12 nu^2) per Newton step
    flops = float(np.sum(np.maximum(r["iterations"] - 1, 0))) * (2.0 / 3.0 * nu ** 3 + 12.0 * nu ** 2)
    tflops = flops * args.steps / dt / 1e12
    peak = P.fp64_peak_tflops(dev)
    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.oracle import OracleAc, OracleContext
        oac = OracleAc(OracleContext(text))
        cores = os.cpu_count() or 1
        m = min(len(cg), max(cores * (K + 1), 4000))
        t0 = time.perf_counter()
        oac.cases(genomes, 3, 2, cg[:m], ck[:m], threads=cores, loading=False)
        m = int(min(len(cg), max(m, m * 3.0 / max(time.perf_counter() - t0, 1e-6))))  # ~3 s sample
        t0 = time.perf_counter()
        oac.cases(genomes, 3, 2, cg[:m], ck[:m], threads=cores, loading=False)
        cdt = time.perf_counter() - t0
        base = {"value": m / cdt / (K + 1), "unit": "topologies/s", "cores": cores, "kind": "port",
                "sample": f"{m} AcNetwork::run_case solves of the same topologies (oracle restatement of "
                          f"ac_validator.cpp) on {cores} threads, {cdt:.1f} s"}
    if rank == 0:
        line = {"metric": "AC N-1 validated topologies/sec", "value": value, "unit": "topologies/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic genomes (seeded, valid), grid as named",
                "config": {"workload": AC_CONFIGS[cfgname]["workload"], "topologies_per_step": n_gen,
                           "cases_per_step": n_gen * (K + 1), "n_buses": grid.n_nodes, "n_contingencies": K,
                           "dense_unknowns_max": nu, "context_setup_s": setup_s,
                           "converged_fraction": float(np.mean(r["converged"])),
                           "mean_iterations": float(np.mean(r["iterations"])),
                           "accepted": int(np.sum(acc)), "l2": "inputs are genomes (KB); no flush needed"},
                "gpu_launches": int(launches),
                "roofline": {"bound": "fp64", "kernel": "k_ac_case (one CTA per case: Newton-Raphson, dense LU)",
                             "achieved": tflops, "peak": peak, "unit": "TFLOP/s",
                             "frac": tflops / peak if peak else None, "traffic": None,
                             "algorithmic": "per Newton step of every case 2/3 nu^3 (partial-pivot LU) + 12 nu^2 "
                                            "(injections, Jacobian), nu = 2 (buses - 1); / the step time",
                             "note": "latency-bound: the LU of a few-dozen-unknown Jacobian is a chain of "
                                     "CTA barriers; the throughput comes from thousands of cases in flight"},
                "e2e": {"value": value, "unit": "topologies/s", "h2d_bytes_per_step": int(genomes.nbytes),
                        "d2h_bytes_per_step": int(n_gen * (4 + 1 + 8)),
                        "call": "tg_ac_full_validation (AcValidator::full_validation for the batch) on host buffers"},
                "clocks": clk.summary()}
        if base is not None:
            line["cpu_baseline"] = base
        print(json.dumps(line), flush=True)


def run_import(args, world, rank):
    """Import stage: build_action_set (importer.cpp:42-70, 239-356) of the
    config's grid with the bridge passes and the split islanding validation on the GPU
    (tg_actionset_build_device), against the same algorithm on the host cores."""
    if rank != 0:
        return
    import paper_2605_10128_b200 as P
    cfgname = args.config if args.config in CONFIGS else "cfg4"
    text = grid_text(cfgname)
    grid = P.grid_from_json_text(text)
    P.build_action_set(grid, device=0)  # warm-up (context, module load)
    times = []
    for _ in range(max(args.steps, 1)):
        t0 = time.perf_counter()
        acts = P.build_action_set(grid, device=0)
        times.append(time.perf_counter() - t0)
    dev_s = statistics.median(times)
    t0 = time.perf_counter()
    host = P.build_action_set(grid)
    host_s = time.perf_counter() - t0
    same = (host.n_actions == acts.n_actions and host.groups == acts.groups
            and host.disconnectables.tolist() == acts.disconnectables.tolist())
    line = {"metric": "action-set import time", "value": dev_s, "unit": "s", "n_gpus": 1, "steps": len(times),
            "warmup": 1, "ms_per_step": 1000 * dev_s, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic grid as named",
            "config": {"workload": CONFIGS[cfgname]["workload"] + "; build_action_set only",
                       "n_actions": acts.n_actions, "n_disconnectables": len(acts.disconnectables),
                       "identical_to_host": bool(same)},
            "gpu_launches": 2,
            "cpu_baseline": {"value": host_s, "unit": "s", "cores": os.cpu_count() or 1, "kind": "port",
                             "sample": "the same build_action_set on the host (enumerate_disconnectables on one "
                                       "thread as in importer.cpp:42-70, split validation on all threads)"},
            "e2e": {"value": dev_s, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4", choices=sorted(set(CONFIGS) | set(AC_CONFIGS)))
    ap.add_argument("--stage", default="dc", choices=["dc", "ac", "import"],
                    help="dc: the MapElites DC N-1 loop (north_star); ac: the AC validation stage; "
                         "import: build_action_set with the graph passes on the GPU")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rng", default="replay", choices=["replay", "philox"],
                    help="lane RNG: the reference's mt19937_64 stream (default) or counter-based Philox4x32-10")
    ap.add_argument("--mode", default="islands", choices=["islands", "shard"],
                    help="N>1: islands (one population per GPU, archive merge; weak scaling) or shard (one "
                         "population, each GPU evaluates a slice of every generation; strong scaling, archive "
                         "bit-identical to one GPU)")
    ap.add_argument("--merge-every", type=int, default=1,
                    help="island archive merge (NCCL allgather + device merge) every M generations when N>1; 0 = never")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup()
    if args.stage == "ac":
        run_ac(args, world, rank)
        return
    if args.stage == "import":
        run_import(args, world, rank)
        return
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch
    import paper_2605_10128_b200 as P

    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    text = grid_text(args.config)
    B = CONFIGS[args.config]["batch"]
    grid = P.grid_from_json_text(text)
    actions = P.build_action_set(grid)
    t_setup = time.perf_counter()
    ctx = P.DcContext(grid, actions, P.DcConfig(), device=dev)  # DcContext ctor: X, T_base, skip records on device
    setup_s = time.perf_counter() - t_setup
    info = ctx.info()
    # islands: one population per rank (seed 1 + rank); shard: one population (seed 1)
    cfg = P.QdConfig(batch_size=B, iters_per_epoch=1 << 30, seed=1 + (rank if args.mode == "islands" else 0),
                     rng=args.rng)
    sess = P.QdSession(ctx, cfg)
    stream = torch.cuda.ExternalStream(P.context_stream(ctx), device=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    ex = None
    shard = None
    # the engine's own NCCL communicator (tg_islands_*) on NCCL runs; the
    # torch.distributed exchange for gloo (ranks sharing a GPU) or on request
    native = False
    if world > 1:
        import torch.distributed as dist
        native = dist.get_backend() == "nccl" and not os.environ.get("TGB_TORCH_EXCHANGE")
    if world > 1 and args.mode == "shard":
        if native:
            from paper_2605_10128_b200.islands import NativeIslands
            nat = NativeIslands(sess)

            class _Shard:
                def step(self, n):
                    nat.shard_step(n)
            shard = _Shard()
        else:
            from paper_2605_10128_b200.islands import BatchShard
            shard = BatchShard(sess)
    elif world > 1 and args.merge_every > 0:
        from paper_2605_10128_b200.islands import IslandExchange, NativeIslands
        ex = NativeIslands(sess) if native else IslandExchange(sess)

    def generations(n):
        if shard is not None:
            shard.step(n)
            return
        # n generations of this island; every merge_every-th one ends with the
        # island exchange (pack -> NCCL allgather -> device merge, on the engine stream)
        if ex is None:
            sess.step(n)
            return
        for _ in range(n):
            sess.step(1)
            generations.count += 1
            if generations.count % args.merge_every == 0:
                ex.exchange()
    generations.count = 0

    # warm-up generations
    generations(args.warmup)
    torch.cuda.synchronize()
    barrier()

    # ---- timed region: exactly K generations, device time, max over ranks
    launches0 = ctx.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        barrier()
        clk.mark()
        e0.record(stream)
        generations(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.kernel_launches() - launches0
    ms = max_over_ranks(ms, world, dev)
    total = B * args.steps * (world if shard is None else 1)  # shard: the ranks share one batch
    value = total / (ms / 1000.0)
    snap = sess.fetch()

    # ---- live roofline of the fused sweep (same loop, sweep bracketed by events)
    P.sweep_timing(ctx, True)
    P.sweep_rows(ctx)  # reset the skip counters
    P.sweep_chunks(ctx)
    flops = 0.0
    E, Ks, Kp = info["n_branches"], info["n_single"], info["k_padded"]
    T = int(json.loads(text).get("timesteps", {}).get("count", 1))
    n_prof = 5
    isl = 0
    r_all = np.zeros(0, np.int64)
    for _ in range(n_prof):
        sess.step(1)
        r = P.batch_ranks(ctx, B)
        live = r[r >= 0]
        r_all = np.concatenate([r_all, live.astype(np.int64)])
        isl += int((r < 0).sum())
        flops += float(E) * Ks * float(np.sum(2.0 * T + 2.0 * live))
    sweep_ms, sweep_n = P.sweep_timing(ctx, False)
    rows_done, rows_offered, rows_overloaded, rows_partial = P.sweep_rows(ctx)
    chunk_tests, chunk_hot = P.sweep_chunks(ctx)
    torch.cuda.synchronize()
    avg_ms = sweep_ms / max(sweep_n, 1)  # one sweep launch (one per timestep per generation)
    step_sweep_ms = sweep_ms / n_prof
    computed_frac = rows_done / rows_offered if rows_offered else 1.0
    partial_frac = rows_partial / rows_offered if rows_offered else 1.0
    dense_tflops = flops / n_prof / (step_sweep_ms * 1e-3) / 1e12
    mean_rank = float(flops / n_prof / (E * Ks) / B / 2.0 - T) if B else 0.0
    # executed FP64 work: blocks past the per-row bound run the first FMA
    # (f_c + T alpha), blocks past the per-element bound also the R FMAs of L R';
    # skipped work cannot change any score
    # executed FP64 work per launch: computed blocks x 128 elements x (2 + 2r),
    # plus the row bound (2 + 2r flops) of every row of a hot chunk
    per_launch = n_prof * T
    executed_flops = (rows_done * 128.0 * (2.0 + 2.0 * mean_rank) + chunk_hot * 32.0 * (2.0 + 2.0 * mean_rank)) / per_launch
    executed_tflops = executed_flops / (avg_ms * 1e-3) / 1e12 if avg_ms else 0.0
    # SURVEY.md 8(d) compulsory bytes per sweep launch: T_base read once
    # (8 E K), every swept candidate's per-candidate vectors in (8 (E + K)(T + r)
    # with T = 1 per launch) and its folded outputs out (8 (E + K): fmax per
    # branch, energy per contingency)
    n_swept = len(r_all) / n_prof
    r_mean = float(np.mean(np.maximum(r_all, 0))) if len(r_all) else 0.0
    alg_bytes = 8.0 * E * Ks + n_swept * 8.0 * (E + Ks) * (1.0 + r_mean) + n_swept * 8.0 * (E + Ks)
    hbm_gbs = alg_bytes / (avg_ms * 1e-3) / 1e9 if avg_ms else 0.0
    # bytes the chunked sweep stages through L2 / shared memory per launch
    # (mostly L2 hits: ncu DRAM traffic is the `traffic` figure)
    stride_mean = float(np.mean((np.maximum(r_all, 0) + 2) & ~1)) if len(r_all) else 2.0
    nch = (E + 31) // 32
    staged_bytes = (n_swept * (8.0 * stride_mean * Kp + nch * 32.0) + (Kp // 128) * nch * 48.0
                    + chunk_hot / per_launch * 32.0 * (8.0 * stride_mean + 8.0 + 48.0))
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        hbm_peak = 7700.0
        hbm_src = "B200_PROFILING.md fallback"
    peak = P.fp64_peak_tflops(dev)
    traffic = None
    ncu = {}
    prof_json = os.path.join(ROOT, "profiles", "sweep_ncu_summary.json")
    if os.path.exists(prof_json):
        try:
            ncu = json.load(open(prof_json)).get(args.config, {})
            traffic = ncu.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            ncu = {}

    # ---- end to end through the reference-facing call with pinned host buffers
    #      (DcContext::evaluate_batch: H2D genomes, evaluate, D2H scores each step)
    rng = np.random.default_rng(7 + rank)
    pool = np.array([e.genome.action_slots + e.genome.disconnection_slots for e in snap.entries], np.int32)
    e2e_steps = max(3, min(args.steps, 10))
    # a distinct batch of mutated archive genomes per timed step (each step
    # copies its own genomes host -> device and its scores device -> host)
    batches = []
    for k in range(e2e_steps + 2):
        parents = pool[rng.integers(0, len(pool), B)]
        batches.append(P.mutate_lanes(ctx, cfg, parents, rng.integers(1, 2 ** 62, B, dtype=np.uint64)))
    g_pin = torch.from_numpy(np.stack(batches).reshape(-1)).pin_memory()
    per = B * (cfg.n_a + cfg.n_d)
    wk = ctx.config.worst_k
    outs = {k: torch.zeros(B * m, dtype=t).pin_memory() for k, t, m in [
        ("lambda_o", torch.float64, 1), ("lambda_c", torch.int32, 1), ("lambda_c0", torch.int32, 1),
        ("lambda_b", torch.float64, 1), ("lambda_d", torch.int32, 1), ("lambda_s", torch.int32, 1),
        ("lambda_r", torch.int32, 1), ("fitness", torch.float64, 1), ("islanded", torch.uint8, 1),
        ("worst_idx", torch.int32, wk), ("worst_energy", torch.float64, wk), ("worst_n", torch.int32, 1),
        ("islanded_outages", torch.int32, 1), ("islanded_busbar_outages", torch.int32, 1)]}
    import ctypes as C
    sc = P.api.L.ScoresC(*[C.cast(C.c_void_p(outs[f].data_ptr()), t) for f, t in P.api.L.ScoresC._fields_])
    d2h = sum(v.numel() * v.element_size() for v in outs.values())
    h2d = per * 4
    for k in range(2):
        P.evaluate_raw(ctx, g_pin.data_ptr() + (e2e_steps + k) * per * 4, B, 3, 2, sc)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        P.evaluate_raw(ctx, g_pin.data_ptr() + k * per * 4, B, 3, 2, sc)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    e2e_s = max_over_ranks(e2e_s, world, dev)
    e2e_value = B * e2e_steps * world / e2e_s

    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(text, B)

    work_bytes = B * (E * 64 + info["k_padded"] * 64)  # per-step candidate rows (feat + contingency rows)
    if rank == 0:
        line = {
            "metric": "N-1-evaluated topologies/sec (DC)", "value": value, "unit": "topologies/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if shard is not None else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic grid (seeded generator tools/synth_grid.py, reference JSON); genomes from the "
                    "device MapElites loop",
            "config": {"workload": CONFIGS[args.config]["workload"], "batch_per_gpu": B,
                       "n_nodes": info["n_nodes"], "n_branches": E, "n_contingencies": info["n_contingencies"],
                       "n_actions": info["n_actions"], "n_disconnectables": info["n_disconnectables"],
                       "parallelism": (f"batch shard x{world}: one population, each rank evaluates {B // world} "
                                       "lanes per generation, NCCL allgather of score slices, every rank inserts "
                                       "all lanes (archive identical to one GPU)" if shard is not None else
                                       f"islands x{world} (seed 1+rank), archives merged every {args.merge_every} "
                                       "generation(s): NCCL allgather of archive blobs + device Repertoire merge"
                                       if ex is not None else f"islands x{world} (seed 1+rank)")
                                      + ("; exchange: engine-native NCCL communicator (tg_islands_*)" if native else
                                         "; exchange: torch.distributed" if world > 1 else ""),
                       "l2": f"per-step candidate working set {work_bytes / 2**20:.0f} MiB > 126 MiB L2 "
                             "(no flush needed)",
                       "step": "one MapElites generation: mutate/crossover + full N-1 evaluation + archive insert",
                       "rng": args.rng,
                       "archive_entries": len(snap.entries), "best_fitness": snap.best_fitness,
                       "context_setup_s": setup_s},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm",
                         "kernel": ("k_sweep_chunked (fused N-1 sweep, scores-only)" if T == 1 else
                                    "mask pass + k_sweep_masked (timestep screening, 8 profiles per launch); "
                                    "bytes per profile"),
                         "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": hbm_gbs / hbm_peak if hbm_peak else None, "traffic": traffic,
                         "algorithmic": "SURVEY.md 8(d) compulsory bytes per launch: 8*E*K (T_base once) + per "
                                        "swept candidate 8*(E+K)*(1+r) in (candidate flows + low-rank factors) "
                                        "and 8*(E+K) out (folded maxima, energies); / the average launch time "
                                        "measured live with CUDA events on the engine stream",
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_ms, "mean_rank": mean_rank,
                         "timesteps": T, "peak_source": hbm_src,
                         "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of one "
                                           "launch (profiles/sweep_ncu_summary.json)",
                         "note": "latency / issue-bound (ncu: issue active ~42 %, warps active ~25 %): the "
                                 "work is the chunk and row bounds plus the exact path of the few overloaded "
                                 "blocks; skipped work provably cannot change a score (tests/test_gpu_scale.py: "
                                 "bit-identical to the dense sweep)",
                         "fp64_executed": {"tflops": executed_tflops, "peak": peak,
                                           "frac": executed_tflops / peak if peak else None,
                                           "flops_per_launch": executed_flops,
                                           "peak_source": "DFMA microbenchmark on this GPU in this run "
                                                          "(MEASURED_PEAKS.json has no FP64 figure)",
                                           "what": "FP64 flops executed: every (row, 128-contingency tile) block "
                                                   "no bound proves safe x 128 x (2 + 2r), plus the row bound "
                                                   "(2 + 2r) of every row of a hot chunk"},
                         "staged_bytes_per_launch": staged_bytes,
                         "dense_equivalent": {"tflops": dense_tflops, "x_fp64_peak": dense_tflops / peak if peak else None,
                                              "flops_per_launch": flops / n_prof / T,
                                              "what": "SURVEY.md 8(d) E*K_single*(2T+2r) per swept candidate / the "
                                                      "launch time: the work of a sweep that evaluates every element "
                                                      "(not a roofline: the exact skip never executes most of it)"},
                         "islanded_fraction": isl / (n_prof * B),
                         "skip": {"executed_block_fraction": computed_frac,
                                  "overloaded_block_fraction": rows_overloaded / rows_offered if rows_offered else 0.0,
                                  "chunk_tests": chunk_tests / per_launch,
                                  "hot_chunk_fraction": chunk_hot / chunk_tests if chunk_tests else None},
                         "ncu": ncu or None},
            "e2e": {"value": e2e_value, "unit": "topologies/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "call": "tg_evaluate_batch (DcContext::evaluate_batch) on pinned host buffers"},
            "clocks": clk.summary(),
        }
        if base is not None:
            line["cpu_baseline"] = base
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
