"""CPU: host-side logic — the circuit/ansatz/observable helpers (a mirror of
circuit.cpp / statevec.cpp), batch sharding, and the data-parallel reduction
with world_size 2 over gloo."""
import os

import numpy as np
import pytest

from paper_2603_02804_b200 import circuits as C
from paper_2603_02804_b200.parallel import combine_partials, shard_range


def test_helpers_bit_exact_vs_oracle(oracle):
    for n, l in [(2, 1), (3, 2), (5, 3), (20, 2)]:
        g, np_ = C.build_hea(n, l)
        g2, np2 = oracle.build_hea(n, l)
        assert np_ == np2 and np.array_equal(g.view(np.uint8), g2.view(np.uint8))
    assert np.array_equal(C.random_parameters(100, 1235), oracle.random_parameters(100, 1235))
    # fp64: numpy's vectorised log/cos may differ from glibc in the last ulp
    np.testing.assert_allclose(C.new_random_state(6, 3, 1234, np.float64),
                               oracle.random_state(6, 3, 1234), rtol=0, atol=1e-15)
    for n in (1, 4, 7, 20):
        lab = C.repeated_ixyz_label(n)
        assert lab == oracle.repeated_ixyz(n)
        assert C.parse_pauli(lab) == oracle.parse_pauli(lab)


def test_helpers_vs_reference(ref):
    g, npar = C.build_hea(6, 4)
    g2, _ = ref.build_hea(6, 4)
    assert np.array_equal(g.view(np.uint8), g2.view(np.uint8))
    assert np.array_equal(C.new_random_state(7, 2, 99), ref.random_state(7, 2, 99, np.float32))
    assert C.parse_pauli("XYZI") == ref.parse_pauli("XYZI")


def test_helper_errors():
    with pytest.raises(ValueError):
        C.build_hea(1, 1)
    with pytest.raises(ValueError):
        C.build_hea(3, 0)
    with pytest.raises(ValueError):
        C.parse_pauli("IXQ")
    with pytest.raises(ValueError):
        C.parse_pauli("")
    with pytest.raises(ValueError):
        C.parse_pauli("IX", 3)


def test_random_state_slices_are_the_global_stream():
    full = C.new_random_state(5, 6, 1234)
    # device generator contract: sample s of the slice starting at first == sample first+s
    from paper_2603_02804_b200.circuits import splitmix_draws
    z = splitmix_draws(1234, 2 * 3 * 32, 64)
    u1 = ((z[0::2] >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    t = 2.0 * np.pi * ((z[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
    re, im = r * np.cos(t), r * np.sin(t)
    inv = 1 / np.sqrt(np.sum(re * re + im * im))
    np.testing.assert_allclose(full[3, :, 0], (re * inv).astype(np.float32), atol=1e-7)


@pytest.mark.parametrize("batch,world", [(1000, 8), (1024, 8), (7, 3), (3, 4), (125, 1)])
def test_shard_range_partitions(batch, world):
    ranges = [shard_range(batch, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == batch
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def _dp_worker(rank, world, port, out):
    import torch.distributed as dist
    import torch
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracles import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    n, layers, batch = 5, 2, 7
    gates, npar = C.build_hea(n, layers)
    theta = C.random_parameters(npar, 1235)
    pauli = C.parse_pauli(C.repeated_ixyz_label(n))
    a, b = shard_range(batch, rank, world)
    psi = C.new_random_state(n, batch, 1234)[a:b]
    loss, grad, _ = o.gradient(gates, n, npar, psi, theta, pauli)
    buf = torch.tensor(np.concatenate([grad, [loss]]), dtype=torch.float64)
    dist.all_reduce(buf)  # the single exchange of the data-parallel step
    if rank == 0:
        out.put(buf.numpy().tolist())
    dist.destroy_process_group()


def test_data_parallel_allreduce_gloo():
    """world_size 2: per-rank shard gradients all-reduced == full-batch gradient."""
    import multiprocessing as mp
    import socket
    from oracles import Oracle
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = np.array(q.get(timeout=120))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, layers, batch = 5, 2, 7
    gates, npar = C.build_hea(n, layers)
    loss, grad, _ = Oracle().gradient(gates, n, npar, C.new_random_state(n, batch, 1234),
                                      C.random_parameters(npar, 1235),
                                      C.parse_pauli(C.repeated_ixyz_label(n)))
    np.testing.assert_allclose(res[:-1], grad, rtol=1e-12, atol=1e-14)
    assert abs(res[-1] - loss) < 1e-12
    l2, g2 = combine_partials([(loss, grad)])
    assert l2 == loss
