"""The N>1 path on CPU: world_size-2 (and 4) gloo process groups run the same
row-shard planning and all-gather code the NCCL bench uses; each rank's rows
come from the C oracle standing in for the GPU kernel (test infrastructure)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_14398_b200.sharding import block_rows, row_shard


def test_row_shard_partition():
    for N in (16, 64, 4096):
        for world in (1, 2, 3, 4, 6, 8):
            rows = [row_shard(N, world, r) for r in range(world)]
            covered = []
            for b, c in rows:
                covered.extend(range(b, b + c))
            assert covered == list(range(N))
            b = block_rows(N, world)
            assert b & (b - 1) == 0
            for begin, count in rows:
                assert begin % b == 0 or count == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from conftest import Golden

    import oracle
    from paper_2305_14398_b200.sharding import gather_rows, row_shard

    g = Golden()
    flat = g.flat(case)
    N = 1 << flat.n_qubits
    begin, count = row_shard(N, world, rank)
    orc = oracle.Oracle()
    ur, ui = orc.circuit_unitary(flat)  # stand-in for this rank's GPU rows
    local_re = torch.from_numpy(ur[begin:begin + count, 0].copy())
    local_im = torch.from_numpy(ui[begin:begin + count, 0].copy())
    re, im = gather_rows(local_re, local_im, N, world)
    if rank == 0:
        np.save(result_path, np.stack([re.numpy(), im.numpy()]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "qft5"), (2, "dj6"), (4, "entangle6"), (3, "qft4")])
def test_gloo_row_gather_reassembles_psi(tmp_path, golden, world, case):
    out = str(tmp_path / "psi.npy")
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    got = np.load(out)
    re, im = golden.psi(case)
    assert np.array_equal(got[0], re) and np.array_equal(got[1], im)


def _last_json(out: str):
    import json

    for line in reversed(out.strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise AssertionError(f"no JSON line in:\n{out}")


@pytest.mark.parametrize("world", [2, 3])
def test_bench_entry_point_runs_world_ranks_over_gloo(world):
    """`python bench.py --gpus N` re-executes itself under torch.distributed.run with
    N ranks; --dry-run then drives the same rank checks, row_shard and gather_rows
    (all_gather_into_tensor, the call NCCL runs on GPUs) over gloo."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", "--gpus", str(world),
                        "--workload", "qft-12"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    line = _last_json(r.stdout)
    assert line["n_gpus"] == world and line["gathered_ok"] and line["backend"] == "gloo"


def test_bench_refuses_more_gpus_than_visible():
    """--gpus N with fewer visible GPUs fails loudly instead of timing one GPU."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    have = torch.cuda.device_count()
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(max(2, have + 1)), "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stdout + r.stderr
    assert "visible GPUs" in _last_json(r.stdout)["error"]
