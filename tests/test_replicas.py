"""The N > 1 bench path on CPU (world_size 2, gloo): "replicas only" — each
rank builds its own cover, no data-path collective; the job time is the max
over ranks and the whole-job value is N x pairs / that time.
The reference arm runs on rank 0 alone; other ranks exit 0 without output."""
import io
import os
import socket
import sys
from contextlib import redirect_stdout

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, times, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms = bench.max_over_ranks(times[rank], world, device="cpu")
        e2e = bench.max_over_ranks(times[rank] * 3.0, world, device="cpu")
        value = bench.whole_job_value(world, 1e6, ms * 1e-3)
        q.put((rank, ms, e2e, value))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_and_value_gloo():
    world, port = 2, _free_port()
    times = [0.41, 0.47]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, times, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for rank, ms, e2e, value in res:
        assert ms == max(times)                           # slowest replica bounds the job
        assert e2e == pytest.approx(3.0 * max(times))
        assert value == pytest.approx(world * 1e6 / (max(times) * 1e-3))


def test_single_rank_is_identity():
    assert bench.max_over_ranks(0.5, 1) == 0.5
    assert bench.whole_job_value(1, 100.0, 2.0) == 50.0


def test_reference_arm_non_zero_rank_is_silent(monkeypatch):
    monkeypatch.setenv("RANK", "1")
    args = bench.parse(["--impl", "reference", "--gpus", "2"])
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = bench.run_reference(args)
    assert rc == 0 and buf.getvalue() == ""
