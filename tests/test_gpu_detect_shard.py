"""One Detector trace split over ranks on the GPU (ShardedDetectorPass):
each rank runs the fused pass on its contiguous shard and screens it with the
boundary hand-off; together the ranks reproduce the single-pass oracle bit
for bit.  Ranks are processes on cuda:0 joined by gloo (the collective path
is host-side; the driver's GPU tier has one device)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _trace(seed, resets):
    from tests.helpers import random_trace, with_measurements
    from tests.oracle_bind import Oracle

    tr = with_measurements(random_trace(8000 + seed, n_iter=2400, n_seg=3, pp=[2, 4, 8][seed % 3],
                                        dp=4, schedule="1f1b"), Oracle(), noise=0.02, seed=seed)
    tr.reset[:] = 0
    if resets:
        tr.reset[[500, 1190, 1800]] = 1
    return tr


def _worker(rank, world, port, seed, resets, results):
    import torch
    import torch.distributed as dist

    from paper_2605_06374_b200.detect_shard import ShardedDetectorPass

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    tr = _trace(seed, resets)
    sp = ShardedDetectorPass(tr, rank, world, torch.device("cuda", 0))
    sp.detect()
    oc = sp.screen()
    st = sp.pass_.status.cpu().numpy()
    ms = sp.pass_.makespan.cpu().numpy()
    results[rank] = (sp.bounds[rank], st.tobytes(), ms.tobytes(), oc.tobytes())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,seed,resets", [(2, 0, False), (3, 1, True), (3, 2, False)])
def test_sharded_trace_equals_single_pass(world, seed, resets, oracle, cuda_device):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    results = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, seed, resets, results), nprocs=world, join=True)
    tr = _trace(seed, resets)
    oms, ost, *_ = oracle.detect(tr)
    ooc, _ = oracle.screen(tr.observed, ost, reset=tr.reset)
    n = tr.n_iter
    st, ms, oc = np.zeros(n, np.uint8), np.zeros(n), np.zeros(n, np.uint8)
    for r in range(world):
        (a, b), s_, m_, o_ = results[r]
        st[a:b] = np.frombuffer(s_, np.uint8)
        ms[a:b] = np.frombuffer(m_, np.float64)
        oc[a:b] = np.frombuffer(o_, np.uint8)
    np.testing.assert_array_equal(st, ost)
    np.testing.assert_array_equal(ms.view(np.uint64), oms.view(np.uint64))
    np.testing.assert_array_equal(oc, ooc)
