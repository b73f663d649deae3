"""Multi-GPU paths (need >= 2 visible GPUs; skipped on a one-GPU box): the
sharded re-plan search finished by the C-ABI collective rh_minloc_allreduce
(NCCL all-gather of (score, index) pairs + device min-loc) and by
torch.distributed (search.distributed_best) give the single-GPU full-space
winner on every rank."""

import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, name, results):
    import torch
    import torch.distributed as dist

    from paper_2605_06374_b200.replan_scenarios import replan_problem
    from paper_2605_06374_b200.search import NcclComm, ReplanSearch, distributed_best

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    *_, inputs = replan_problem(name)
    s = ReplanSearch(inputs, dev)
    a, b = s.shard(rank, world)
    best, idx = s.eval_async(a, b)
    comm = NcclComm(rank, world, dev)
    comm.minloc(best, idx)
    torch.cuda.synchronize()
    c_abi = (float(best.item()), int(idx.item()))
    comm.close()
    via_torch = distributed_best(s)
    results[rank] = (c_abi, via_torch)
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_sharded_search_collectives(name, cuda_device):
    import torch
    import torch.multiprocessing as mp

    world = torch.cuda.device_count()
    if world < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2605_06374_b200.replan_scenarios import replan_problem
    from paper_2605_06374_b200.search import ReplanSearch

    *_, inputs = replan_problem(name)
    full = ReplanSearch(inputs).best()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    results = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, name, results), nprocs=world, join=True)
    for r in range(world):
        c_abi, via_torch = results[r]
        assert c_abi == full and tuple(via_torch) == full, (r, c_abi, via_torch, full)
