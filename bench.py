#!/usr/bin/env python
"""Benchmark: interactions/sec of the device reduction loop (BASELINE.json).

Default workload (``--workload batch``): 4096 independent Ackermann(3,6) nets
(BASELINE.json configs[4]), sharded contiguously over the ranks of a torchrun
job (one GPU per rank, no data-path collective: ``scaling: strong`` — the total
batch is fixed). A step reduces every net of the shard to normal form in one
persistent-kernel launch. ``value`` = all nets' interactions / max-over-ranks
device time (CUDA events around the launch, inputs resident in HBM, L2 flushed
between steps). ``e2e`` = the same metric through the C ABI with host buffers:
load (H2D), reduce, D2H of the results and the native host finalize, per step.

Single-net configurations (A(3,10), A(3,8), fib(18)) are measured once each on
rank 0 after the timed batch and reported under ``single_nets``; they do not
shard (replicas only).

``--impl reference`` times the reference algorithm on the host cores instead:
the C++ restatement in oracle/ (the reference package is pure Python and
cannot travel to the GPU box), with every host thread, on bounded samples.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the reference package `inet` (net builders, value oracles) from baseline/_ref
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))

BATCH_NETS = 4096
BATCH_PARAMS = (3, 6)
GOLDEN_A36 = 344_964  # SURVEY.md §8(c), pinned by tests/test_oracle.py
SINGLE = {
    "A(3,10)": ("ackermann", (3, 10), 89_404_824),
    "A(3,8)": ("ackermann", (3, 8), 5_574_030),
    "fib(18)": ("fibonacci", (18,), 50_515),
    # the wide L-system net (130K redexes in its widest
    # loop), where throughput rather than span binds; runs on the whole GPU
    "lsystem(26)": ("lsystem", (26,), 1_028_428),
}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region.

    NVML (pynvml) every 10 ms from a thread, with one sample at entry and one at
    exit so even a short region is covered; nvidia-smi -lms as the fallback.
    """

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.nvml = None
        self.samples: list[tuple[float, float, int]] = []  # (sm MHz, max sm MHz, reason bits)
        self.lines: list[str] = []
        self.stop = threading.Event()

    def _nvml_sample(self):
        n = self.nvml
        sm = n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(self.handle, n.NVML_CLOCK_SM)
        try:
            bits = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        except AttributeError:
            bits = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle)
        self.samples.append((float(sm), float(mx), int(bits)))

    def _nvml_loop(self):
        while not self.stop.wait(0.01):
            try:
                self._nvml_sample()
            except Exception:  # noqa: BLE001 - sampling must never break the benchmark
                return

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            # CUDA ordinal -> NVML index (CUDA_VISIBLE_DEVICES may remap)
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].isdigit() else self.gpu
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nvml_sample()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.t.join(timeout=1)
            try:
                self._nvml_sample()
            except Exception:  # noqa: BLE001
                pass
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        for s, m, bits in self.samples:
            sm.append(s)
            mx.append(m)
            for name, bit in self.REASONS.items():
                if bits & bit:
                    reasons.add(name)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


# ---------------------------------------------------------------------------
# algorithmic bytes: agent = 4 B label + 4 B per port,
# equation = 8 B; interaction reads its equation and both agents and writes the
# rhs equations and new agents; a communication merge moves 24 B.


def rule_bytes(rules) -> list[int]:
    from paper_1404_0076_b200.flat import is_var

    out = []
    for rule in rules.rules.values():
        rd = 8 + (4 + 4 * rule.lhs_a.arity) + (4 + 4 * rule.lhs_b.arity)
        wr = 8 * len(rule.rhs)
        for e in rule.rhs:
            for side in (e.lhs, e.rhs):
                work = [side]
                while work:
                    t = work.pop()
                    if not is_var(t):
                        wr += 4 + 4 * t.sym.arity
                        work.extend(t.children)
        out.append(rd + wr)
    return out


def algorithmic_bytes(rules, rule_counts, communications) -> int:
    per = rule_bytes(rules)
    return int(sum(int(c) * b for c, b in zip(rule_counts, per)) + 24 * int(communications))


# ---------------------------------------------------------------------------


def load_peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic(workload: str):
    """dram bytes per launch from the committed ncu capture (profiles/), if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(workload)
    except (OSError, ValueError):
        return None


def ncu_issue(workload: str):
    """Instruction-issue figures of the workload's timed kernel(s) from the committed
    ncu capture (profiles/issue.json, tools/ncu_issue.py): what binds these kernels
    is issue and latency, not HBM."""
    try:
        with open(os.path.join(ROOT, "profiles", "issue.json")) as fh:
            rec = json.load(fh).get(workload)
    except (OSError, ValueError):
        return None
    if rec is None:
        return None
    keep = ("issue_active_pct_of_active_smsp", "lanes_active_avg", "thread_inst_per_interaction", "warp_inst",
            "duration_ns", "kernels", "source")
    return {k: rec[k] for k in keep if k in rec}


def cpu_sample(program_name: str, params, seconds: float, threads: int) -> dict:
    """Time the oracle (reference algorithm, C++ port) on the host for ~seconds."""
    from oracle import oracle as O
    from inet.bench import program

    prog = program(program_name)
    rules = O.rules_for(program_name)
    net = prog.build_input(*params)
    deadline = time.perf_counter() + seconds
    done = [0] * threads
    ints = [0] * threads

    def worker(k):
        while time.perf_counter() < deadline or done[k] == 0:
            r = O.run_config(net, rules, collect=False)
            done[k] += 1
            ints[k] += r.interactions

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        list(ex.map(worker, range(threads)))
    wall = time.perf_counter() - t0
    return {"value": sum(ints) / wall, "nets": sum(done), "wall_s": wall, "interactions": sum(ints)}


def _py_reference_net(params):
    """One net through the reference's own Python reducer (baseline/_ref), in a worker process."""
    sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
    from inet.bench import program
    from inet.engine import EngineConfig, evaluate

    prog = program("ackermann")
    t0 = time.perf_counter()
    r = evaluate(prog.build_input(*params), prog.rules, EngineConfig(collect_stats=False))
    return r.total_interactions, time.perf_counter() - t0


def python_reference_sample(seconds: float, threads: int, params=(3, 5)) -> dict:
    """The unmodified Python reference (inet.engine.evaluate from baseline/_ref) on all host
    cores, one net per process (multiprocessing, as BASELINE.md §2 plans), for ~seconds."""
    import multiprocessing as mp

    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "inet")):
        return {"unavailable": "baseline/_ref not installed"}
    ctx = mp.get_context("spawn")
    ints, nets = 0, 0
    t0 = time.perf_counter()
    with ctx.Pool(threads) as pool:
        pending = [pool.apply_async(_py_reference_net, (params,)) for _ in range(threads)]
        while pending:
            r = pending.pop(0).get()
            ints += r[0]
            nets += 1
            if time.perf_counter() - t0 < seconds:
                pending.append(pool.apply_async(_py_reference_net, (params,)))
    wall = time.perf_counter() - t0
    return {"value": ints / wall, "unit": "interactions/s", "cores": threads, "kind": "reference",
            "sample": f"{nets} nets of ackermann{params} in {wall:.1f}s through inet.engine.evaluate "
                      f"(the unmodified Python reference, baseline/_ref), one net per process"}


def run_reference(args) -> None:
    rank, _, world = dist_env()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    name, params, wl = workload_spec(args.workload)
    per_step = []
    for i in range(args.warmup + args.steps):
        s = cpu_sample(name, params, args.ref_seconds, threads)
        if i >= args.warmup:
            per_step.append(s)
    total_i = sum(s["interactions"] for s in per_step)
    total_t = sum(s["wall_s"] for s in per_step)
    value = total_i / total_t
    line = {
        "impl": "reference",
        "metric": "interactions/sec",
        "value": value,
        "unit": "interactions/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000 * total_t / len(per_step),
        "higher_is_better": True,
        "scaling": "strong" if args.workload == "batch" else "replicas",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (deterministic Ackermann/Fibonacci nets, no RNG)",
        "config": wl,
        "cpu_baseline": {
            "value": value,
            "unit": "interactions/s",
            "cores": threads,
            "kind": "port",
            "sample": f"{sum(s['nets'] for s in per_step)} nets of {name}{params} over {args.steps} steps of "
                      f"~{args.ref_seconds}s, oracle/inet_oracle.cpp (C++ restatement of "
                      f"inet.engine.evaluate), one net per host thread; a rate measured on a bounded sample "
                      f"of the workload (each step a slice of the {wl.get('nets', 1)} nets), not a full pass",
            "extrapolated": "rate over the sampled nets; every net of the workload is identical",
        },
        "e2e": {"value": value, "unit": "interactions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_python_reference:
        # the reference's own Python reducer beside the C++ port
        line["python_reference"] = python_reference_sample(args.py_ref_seconds, threads)
    print(json.dumps(line), flush=True)


def workload_spec(name: str):
    if name == "batch":
        return "ackermann", BATCH_PARAMS, {"workload": f"batch {BATCH_NETS} x Ackermann(3,6)", "nets": BATCH_NETS,
                                           "net": "A(3,6)", "l2": "flushed between steps (256 MiB write)"}
    prog, params, _ = SINGLE[{"a310": "A(3,10)", "a38": "A(3,8)", "fib18": "fib(18)"}[name]]
    label = {"a310": "A(3,10)", "a38": "A(3,8)", "fib18": "fib(18)"}[name]
    return prog, params, {"workload": f"single net {label}", "nets": 1, "net": label,
                          "l2": "flushed between steps (256 MiB write)"}


def nat_text(height: int) -> str:
    """print_configuration of the normal form S^height(Z) (lang.py:371-396)."""
    return "net " + "S(" * height + "Z" + ")" * height + " : ;"


def timed_outcomes(ctx, prep, n_nets: int, height: int) -> list:
    """(interactions, text sha prefix) of every net of the last launch, each text checked."""
    from paper_1404_0076_b200 import engine, shard

    ctx.finalize(0xFFFFFFFF, 0)
    tab = engine.label_table(prep.labels)
    want = nat_text(height)
    out = []
    for i in range(n_nets):
        text = ctx.text(i, tab)
        assert text == want, (i, text[:80])
        out.append(shard.outcome(ctx.stats(i).interactions, text))
    return out


def check_normal_forms(ctx, n_nets: int, height: int, sample: int = 64) -> None:
    """Every sampled net must reduce to S^height(Z) with no residual equation."""
    ctx.finalize(0xFFFFFFFF, 0)
    step = max(1, n_nets // sample)
    for i in range(0, n_nets, step):
        agents, iface, eqs = ctx.result(i)
        assert len(eqs) == 0 and len(iface) == 1 and len(agents) == height + 1, (i, len(agents), len(eqs))


def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1404_0076_b200 import EngineConfig, _native, engine, shard
    from inet.bench import ackermann_value, fibonacci_value, program

    rank, local, world = dist_env()
    if world > 1:
        # --test-one-device: every rank on GPU 0 over gloo (exercises the multi-rank
        # path on a one-GPU box; NCCL refuses two ranks on one device)
        dist.init_process_group("gloo" if args.test_one_device else "nccl", init_method="env://")
    dev = 0 if args.test_one_device else local
    torch.cuda.set_device(dev)
    cdev = "cpu" if args.test_one_device else f"cuda:{dev}"  # where the control collectives run
    name, params, wl = workload_spec(args.workload)
    prog = program(name)
    if args.workload == "batch":
        lo, hi = shard.shard_bounds(BATCH_NETS, world, rank)
        configs = [prog.build_input(*params) for _ in range(hi - lo)]
        per_net = GOLDEN_A36
    else:
        configs = [prog.build_input(*params)]
        per_net = SINGLE[wl["net"]][2]
    n_nets = len(configs)
    ecfg = EngineConfig(collect_stats=False, threads=args.threads, device=dev)
    prep = engine.prepare(configs, prog.rules)
    ctx = _native.Context(dev)
    ctx.load_rules(prep.blob)
    ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
    k = engine.native_cfg(ecfg)
    k.count_rules = 1
    code, _ = ctx.reduce(k)  # accounting + correctness run
    assert code == _native.OK, _native.strerror(code)
    ti, tc, max_rounds, nfail = ctx.totals()
    assert nfail == 0 and ti == per_net * n_nets, (ti, per_net * n_nets)
    counts = np.zeros(len(prog.rules.rules), dtype=np.uint64)
    for i in range(n_nets):
        counts += ctx.rule_counts(i, len(prog.rules.rules))
    alg_bytes = algorithmic_bytes(prog.rules, counts, tc)
    height = ackermann_value(*params) if name == "ackermann" else fibonacci_value(*params)
    check_normal_forms(ctx, n_nets, height)
    k.count_rules = 0

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{dev}")

    def flush_l2():
        flush.zero_()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush_l2()
        ctx.rerun(k)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(dev) as clocks:
        for _ in range(args.steps):
            flush_l2()
            times.append(ctx.rerun(k))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the timed launches' own outcome (the count_rules=0 kernel variant): status and
    # totals of the last timed launch, and every net's printed normal form
    ctx.collect()
    ti_t, tc_t, _mr_t, nfail_t = ctx.totals()
    assert nfail_t == 0 and ti_t == ti and tc_t == tc, (ti_t, tc_t, nfail_t)
    outcomes = timed_outcomes(ctx, prep, n_nets, height)
    my_ms = sum(times)
    max_ms = shard.max_over_ranks(my_ms, device=cdev)
    # interactions of one step, all ranks (each rank verified its own count above)
    total_interactions = int(shard.sum_over_ranks([float(ti)], device=cdev)[0])
    value = total_interactions * args.steps / (max_ms / 1000.0)
    kernel_ms = my_ms / args.steps

    # e2e through the C ABI with host buffers (H2D, kernel, D2H, host finalize)
    e2e_times = []
    h2d = d2h = 0
    for i in range(max(1, args.e2e_steps)):
        t0 = time.perf_counter()
        ctx.load_batch(prep.agents, prep.agent_off, prep.eqs, prep.eq_off, prep.iface, prep.iface_off, prep.n_vars)
        code, _ = ctx.reduce(k)
        ctx.finalize(0xFFFFFFFF, 0)
        agents0, _, _ = ctx.result(0)
        e2e_times.append(time.perf_counter() - t0)
        assert code == _native.OK and len(agents0) == height + 1
        h2d, d2h = ctx.io_bytes()
        assert ctx.totals()[0] == ti
    e2e_max = shard.max_over_ranks(sum(e2e_times), device=cdev)
    e2e_value = total_interactions * len(e2e_times) / e2e_max

    # e2e through the Python API a user calls: evaluate_batch(as_text=True) on
    # this rank's shard — flattening the reference's term objects, H2D, the
    # reduction, D2H, finalize and the canonical text of every net
    api_times = []
    for _ in range(min(args.warmup, 2)):  # untimed: first-touch of the host result buffers
        engine.evaluate_batch(configs, prog.rules, ecfg, as_terms=False, as_text=True)
    for _ in range(max(1, args.api_steps)):
        t0 = time.perf_counter()
        out = engine.evaluate_batch(configs, prog.rules, ecfg, as_terms=False, as_text=True)
        api_times.append(time.perf_counter() - t0)
        assert out.total_interactions == ti
    api_max = shard.max_over_ranks(min(api_times), device=cdev)
    api_value = total_interactions / api_max

    # final result gather: per-net (interactions, text sha) to rank 0
    gathered = shard.gather_outcomes(outcomes, world)
    if rank == 0:
        want = shard.outcome(per_net, nat_text(height))
        assert len(gathered) == (BATCH_NETS if args.workload == "batch" else 1)
        assert all(o == want for o in gathered), "gathered outcomes differ"

    peak, peak_kind = load_peaks()
    achieved = alg_bytes / (kernel_ms / 1000.0) / 1e9
    line = None
    if rank == 0:
        info = ctx.info()
        line = {
            "metric": "interactions/sec",
            "value": value,
            "unit": "interactions/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": max_ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if args.workload == "batch" else "replicas",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic (deterministic Ackermann nets built by the reference builders inet.bench.program, no RNG)",
            "config": dict(wl, parallelism=f"dp{world} (nets sharded, no collective)",
                           interactions_per_net=per_net, rounds_per_net=max_rounds,
                           threads_per_net=engine.native_cfg(ecfg).threads or "auto",
                           tier="SMGCX"[ctx.stats(0).tier], agent_hw=ctx.stats(0).agent_hw,
                           var_hw=ctx.stats(0).var_hw),
            "e2e": {"value": e2e_value, "unit": "interactions/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "C ABI inet_batch_load+inet_batch_reduce+inet_batch_finalize, host flat buffers"},
            "e2e_api": {"value": api_value, "unit": "interactions/s", "ms": 1000 * api_max,
                        "path": "paper_1404_0076_b200.evaluate_batch(configs, rules, as_terms=False, as_text=True): "
                                "flatten + H2D + reduce + D2H + finalize + canonical text, best of "
                                f"{len(api_times)} after {min(args.warmup, 2)} untimed"},
            "gather": {"nets": len(gathered), "bytes_per_net": 24,
                       "what": "per-net (interactions, sha256 prefix of the printed normal form) gathered to "
                               "rank 0 after the timed region; every net checked against S^509(Z)"},
            "gpu_launches": args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(args.workload),
                         "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "issue": ncu_issue(args.workload),
                         "note": "SURVEY.md §8(d) bytes: per-rule (read+write) x device rule histogram "
                                 "+ 24 B per communication"},
            "clocks": clocks.summary(),
            "device": info,
        }
    if world > 1:
        dist.barrier()
    # single nets (rank 0, N=1 headline for A(3,10)); replicas only
    if rank == 0 and args.single:
        singles = {}
        for label, (pname, pparams, golden) in SINGLE.items():
            p = program(pname)
            pr = engine.prepare([p.build_input(*pparams)], p.rules)
            c2 = _native.Context(dev)
            c2.load_rules(pr.blob)
            c2.load_batch(pr.agents, pr.agent_off, pr.eqs, pr.eq_off, pr.iface, pr.iface_off, pr.n_vars)
            kk = engine.native_cfg(EngineConfig(collect_stats=False))
            code, _ = c2.reduce(kk)
            st = c2.stats(0)
            assert code == _native.OK and st.interactions == golden, (label, st.interactions)
            best = []
            for _ in range(5):
                flush_l2()
                best.append(c2.rerun(kk))
            ms = min(best)
            singles[label] = {"interactions": golden, "rounds": st.rounds, "device_ms": ms, "tier": "SMGCXR"[st.tier],
                              "sm_mhz": st.sm_mhz,
                              "agent_hw": st.agent_hw, "var_hw": st.var_hw,
                              "interactions_per_s": golden / (ms / 1000.0),
                              "us_per_round": 1000.0 * ms / max(st.rounds, 1)}
            mode, _ = engine._plan(EngineConfig(collect_stats=False), p.rules, [p.build_input(*pparams)])
            if mode != engine.MODE_FAST:
                # what evaluate() runs by default for this net (reference-exact counts), and tier R
                for key, kr in (("default_path", engine.native_cfg(EngineConfig(collect_stats=False),
                                                                   mode == engine.MODE_R, mode == engine.MODE_STAMPS)),
                                ("reference_order", engine.native_cfg(EngineConfig(collect_stats=False), True))):
                    code, _ = c2.reduce(kr)
                    st_r = c2.stats(0)
                    assert code == _native.OK and st_r.interactions == golden
                    ms_r = min(c2.rerun(kr) for _ in range(3))
                    singles[label][key] = {
                        "device_ms": ms_r, "rounds": st_r.rounds, "communications": int(st_r.communications),
                        "tier": "SMGCXR"[st_r.tier], "interactions_per_s": golden / (ms_r / 1000.0),
                        "us_per_loop": 1000.0 * ms_r / max(st_r.rounds, 1)}
                singles[label]["default_path"]["mode"] = mode
            # end to end through the public API (default evaluation order), host objects in, text out
            e2e = []
            for _ in range(3):
                t0 = time.perf_counter()
                _text, ints, _comms = engine.evaluate_text(p.build_input(*pparams), p.rules)
                e2e.append(time.perf_counter() - t0)
                assert ints == golden
            singles[label]["e2e_ms"] = 1000.0 * min(e2e)
            if label == "A(3,10)":
                singles[label]["issue"] = ncu_issue("a310")
            singles[label]["e2e_path"] = "evaluate_text(config, rules): flatten + H2D + reduce + D2H + finalize + print"
            # the reference's own call: evaluate() returning reference term objects (EvalResult.final)
            t0 = time.perf_counter()
            res = engine.evaluate(p.build_input(*pparams), p.rules, EngineConfig(collect_stats=False))
            singles[label]["evaluate_ms"] = 1000.0 * (time.perf_counter() - t0)
            assert res.total_interactions == golden
            c2.close()
        line["single_nets"] = singles
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        s = cpu_sample(name, params, args.cpu_seconds, threads)
        line["cpu_baseline"] = {
            "value": s["value"], "unit": "interactions/s", "cores": threads, "kind": "port",
            "sample": f"{s['nets']} nets of {name}{params} in {s['wall_s']:.1f}s, oracle/inet_oracle.cpp "
                      f"(C++ restatement of inet.engine.evaluate), one net per host thread",
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=["batch", "a310", "a38", "fib18"], default="batch")
    ap.add_argument("--threads", type=int, default=0, help="CTA size per net (0 = auto)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--api-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-python-reference", action="store_true")
    ap.add_argument("--test-one-device", action="store_true",
                    help="(testing) all ranks on GPU 0 with gloo collectives")
    ap.add_argument("--py-ref-seconds", type=float, default=15.0)
    ap.add_argument("--no-single", dest="single", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
