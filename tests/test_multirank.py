"""World-size-2 gloo run of the batch-sharding host logic (CPU-only).

The GPU work of each rank is independent; what can go wrong across ranks is
the partition (every net exactly once, in order), the max-over-ranks timing
and the gather of per-net outcomes. Each rank here reduces its shard with the
CPU oracle standing in for its device, exactly as bench.py's ranks would.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_nets, out):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1404_0076_b200 import shard
    from inet.bench import program

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard.shard_bounds(n_nets, world, rank)
        prog = program("ackermann")
        rules = O.rules_for("ackermann")
        params = [(2, k % 4) for k in range(n_nets)]
        local = []
        texts = []
        for m, n in params[lo:hi]:
            r = O.run_config(prog.build_input(m, n), rules, collect=False)
            local.append(shard.outcome(r.interactions, r.printed()))  # bench.py's gathered format
            texts.append((m, n, r.printed()))
        t = shard.max_over_ranks(float(rank + 1))
        tot = shard.sum_over_ranks([sum(x[0] for x in local), len(local)])
        allv = list(zip(shard.gather_outcomes(texts, world), shard.gather_outcomes(local, world)))
        if rank == 0:
            out.put((t, tot, allv))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_every_net_once():
    from paper_1404_0076_b200.shard import shard_bounds

    for n in (1, 7, 4096):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_bounds(n, world, r)
                assert hi - lo in (n // world, n // world + 1)
                seen.extend(range(lo, hi))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def test_two_rank_gloo_shard_and_gather():
    world, n_nets = 2, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_nets, q)) for r in range(world)]
    for p in procs:
        p.start()
    t, tot, allv = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0  # max over ranks
    assert tot[1] == n_nets
    assert [(m, n) for (m, n, _), _ in allv] == [(2, k % 4) for k in range(n_nets)]
    from inet.bench import ackermann_value
    from paper_1404_0076_b200 import shard

    for (m, n, text), (ints, sha) in allv:
        assert text.count("S(") == ackermann_value(m, n)
        assert (ints, sha) == shard.outcome(ints, text)
    assert tot[0] == sum(o[0] for _, o in allv)


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu(tmp_path):
    """bench.py under torchrun with 2 ranks (both on GPU 0, gloo control
    collectives): shards, max-over-ranks timing and the final gather of all
    4096 nets' outcomes to rank 0, which checks every one."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--test-one-device", "--no-single", "--no-cpu-baseline",
           "--api-steps", "1", "--e2e-steps", "1"]
    proc = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0, proc.stderr[-3000:]
    line = json.loads([l for l in proc.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["gather"]["nets"] == 4096
    assert line["value"] > 0 and line["e2e"]["value"] > 0
