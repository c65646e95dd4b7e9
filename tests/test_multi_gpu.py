"""The multi-device paths on one B200:

* the NCCL all-gather of psi rows inside libqsb (the in-process multi-device
  handle's path, forced onto a one-rank communicator with QSB_FLAG_NCCL_GATHER),
* the one-process-per-GPU communicator (qsb_comm_create + qsb_plan_allgather_state),
* virtual shards (repeated device ids) under the default stream-K schedule: one
  stream per physical device, so concurrent persistent grids cannot deadlock,
* bench.py refusing a GPU count it cannot honour.
The oracle (C restatement) is the checker only."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2305_14398_b200 as q
from paper_2305_14398_b200 import native
from paper_2305_14398_b200.simulator import B200UnitarySimulator, Comm, nccl_unique_id, nccl_version

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a_re, a_im, b_re, b_im):
    return float(np.sqrt(np.sum((a_re - b_re) ** 2 + (a_im - b_im) ** 2)) / np.sqrt(np.sum(b_re ** 2 + b_im ** 2)))


@pytest.mark.parametrize("name,n", [("qft", 4), ("qft", 7), ("entangle", 10), ("deutsch-jozsa", 9), ("qft", 11)])
def test_nccl_gather_in_host_api(orc, name, n):
    """QSB_FLAG_NCCL_GATHER: psi rows are all-gathered by ncclAllGather into a
    device-resident psi and read back from it — bit-identical to the direct copy."""
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    plain = B200UnitarySimulator(device=0)
    nccl = B200UnitarySimulator(device=0, flags=native.FLAG_NCCL_GATHER)
    a = plain.simulate_full_state(flat)
    b = nccl.simulate_full_state(flat)
    plain.close()
    nccl.close()
    assert np.array_equal(a.re, b.re) and np.array_equal(a.im, b.im)
    re, im = orc.fsv(flat)
    assert rel(b.re, b.im, re, im) <= 1e-10
    assert nccl_version() >= 22000


def test_comm_allgather_one_rank(orc):
    """The multi-process entry points on a one-rank communicator: the all-gathered
    psi equals the plan's own rows."""
    import torch

    c, reg = q.make_named_circuit("qft", 10)
    flat = native.flatten(c, reg)
    N = 1 << 10
    sim = B200UnitarySimulator(device=0)
    comm = Comm(sim, nccl_unique_id(), 1, 0)
    plan = sim.plan(flat)
    plan.execute()
    re = torch.empty(N, dtype=torch.float64, device="cuda")
    im = torch.empty(N, dtype=torch.float64, device="cuda")
    re2 = torch.empty_like(re)
    im2 = torch.empty_like(im)
    plan.allgather_state(comm, re.data_ptr(), im.data_ptr())
    plan.copy_state(re2.data_ptr(), im2.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(re, re2) and torch.equal(im, im2)
    o_re, o_im = orc.fsv(flat)
    assert rel(re.cpu().numpy(), im.cpu().numpy(), o_re, o_im) <= 1e-10
    # the optional U all-gather: the one rank's rows are the whole U
    ur = torch.empty(N * N, dtype=torch.float64, device="cuda")
    ui = torch.empty_like(ur)
    plan.allgather_unitary(comm, ur.data_ptr(), ui.data_ptr())
    torch.cuda.synchronize()
    want = sim.build_unitary(flat)
    assert np.array_equal(ur.cpu().numpy().reshape(N, N), want[0])
    assert np.array_equal(ui.cpu().numpy().reshape(N, N), want[1])
    # a plan that does not own rank 0's block of a 2-rank split is refused
    with pytest.raises(Exception, match="must own rows"):
        half = sim.plan(flat, None, N // 2, N // 2)
        half.allgather_state(comm, re.data_ptr(), im.data_ptr())
    plan.close()
    comm.close()
    sim.close()


def test_virtual_shards_stream_k_no_deadlock():
    """devices = [0, 0, 0, 0] with the default schedule (stream-K at QFT-12's 1024-row
    shards): 20 host calls complete and match one device within 1e-10. Before the
    one-stream-per-device rule the four shards ran on four streams of one GPU."""
    assert "QSB_SPLITK" not in os.environ and "QSB_STREAMK" not in os.environ
    c, reg = q.make_named_circuit("qft", 12)
    flat = native.flatten(c, reg)
    one = B200UnitarySimulator(device=0)
    ref = one.simulate_full_state(flat)
    one.close()
    four = B200UnitarySimulator(devices=[0, 0, 0, 0])
    for _ in range(20):
        out = four.simulate_full_state(flat)
        assert rel(out.re, out.im, ref.re, ref.im) <= 1e-10
    four.close()


def test_bench_gpus_beyond_visible_fails_loudly():
    import torch

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(torch.cuda.device_count() + 1),
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 2, r.stdout + r.stderr


@pytest.mark.parametrize("name,n", [("qft", 5), ("entangle", 10), ("deutsch-jozsa", 11), ("qft", 12)])
def test_sharded_host_call_one_rank(orc, name, n):
    """qsb_simulate_full_state_sharded on a one-rank communicator: the rank's row
    block is all of U, psi comes back through ncclAllGather — bit-identical to the
    single-process call, cold and plan-cached."""
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    plain = B200UnitarySimulator(device=0)
    want = plain.simulate_full_state(flat)
    plain.close()
    for flags in (0, native.FLAG_NO_PLAN_CACHE):
        sim = B200UnitarySimulator(device=0, flags=flags)
        comm = Comm(sim, nccl_unique_id(), 1, 0)
        for _ in range(2):
            got = sim.simulate_full_state_sharded(flat, None, comm)
            assert np.array_equal(got.re, want.re) and np.array_equal(got.im, want.im)
        comm.close()
        sim.close()
