"""The N>1 benchmark path on CPU: world_size-2 gloo process group, the same aggregation bench.py
uses (max over ranks of the device time, sum of agent updates)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_0911_2900_b200.dist import aggregate
    wall, upd = aggregate(0.5 + rank, 1e6 * (rank + 1))
    q.put((rank, wall, upd))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_aggregation_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(90)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    for _, wall, upd in res:
        assert wall == 1.5 and upd == 3e6


def test_single_process_is_identity():
    from paper_0911_2900_b200.dist import aggregate
    assert aggregate(0.25, 123.0) == (0.25, 123.0)


@pytest.mark.timeout(300)
def test_reference_arm_under_torchrun_prints_one_line():
    """bench.py --impl reference launched the driver's way for N=2: rank 0 alone runs the
    reference CPU path and prints one JSON line; rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    import oracle
    if not oracle.have_reference():
        pytest.skip("oracle/_ref not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "corridor"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["warmup"] == 3 and d["steps"] == 3
    assert d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["kind"] == "reference"
