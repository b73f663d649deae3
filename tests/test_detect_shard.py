"""One Detector trace sharded over ranks (paper_2605_06374_b200.detect_shard):
the screen's (series length, visible tail) hand-off across shard boundaries
reproduces the single-pass DetectorState.observe outcomes bit for bit
(detector.py:198-271).  CPU: gloo ranks with the oracle as the screen."""

import os
import socket

import numpy as np
import pytest

from paper_2605_06374_b200.detect_shard import shard_bounds, tail_state


def _series(seed, n):
    rng = np.random.default_rng(seed)
    base = 10.0 + rng.standard_normal(n) * rng.choice([0.05, 0.5, 2.0])
    if seed % 3 == 0:
        base = np.round(base, 1)  # ties in the median / MAD
    spikes = rng.random(n) < rng.choice([0.05, 0.2, 0.5])
    obs = np.where(spikes, base * rng.uniform(1.1, 3.0, n), base)
    st = (rng.random(n) < 0.3).astype(np.uint8)
    st |= ((rng.random(n) < 0.2).astype(np.uint8) << 1)
    reset = (rng.random(n) < 0.004).astype(np.uint8) if seed % 2 else None
    return obs, st, reset


def _oracle_fn(window, fe=True):
    from tests.oracle_bind import Oracle

    o = Oracle()

    def fn(obs, st, rst, L, hist):
        return o.screen(obs, st, window=window, kappa=3.0, filter_enabled=fe, series_len=L,
                        hist=list(hist), reset=rst)
    return fn


def _worker(rank, world, port, seed, window, align, results):
    import torch.distributed as dist

    from paper_2605_06374_b200.detect_shard import screen_handoff

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    obs, st, reset = _series(seed, 3000 + 117 * seed)
    bounds = shard_bounds(len(obs), world, reset if align else None)
    oc = screen_handoff(obs, st, reset, bounds, rank, _oracle_fn(window), window=window)
    results[rank] = (bounds[rank], oc.tobytes())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,seed,window,align", [
    (2, 0, 20, False), (2, 1, 20, True), (3, 2, 5, False), (3, 3, 33, True), (4, 5, 1, False),
    (4, 7, 64, False)])
def test_sharded_screen_equals_single_pass(world, seed, window, align, oracle):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    results = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, seed, window, align, results), nprocs=world, join=True)
    obs, st, reset = _series(seed, 3000 + 117 * seed)
    full, _ = oracle.screen(obs, st, window=window, reset=reset)
    got = np.zeros(len(obs), np.uint8)
    for r in range(world):
        (a, b), oc = results[r]
        got[a:b] = np.frombuffer(oc, np.uint8)
    np.testing.assert_array_equal(got, full)


def test_tail_state_matches_sequential_series(oracle):
    """The hand-off state derived from the outcome bits equals the state the
    oracle carries: screening the second half from it gives the same bits."""
    for seed in range(6):
        obs, st, reset = _series(seed, 1500)
        for w in (1, 7, 20, 64):
            full, L = oracle.screen(obs, st, window=w, reset=reset)
            c = 700
            first, L1 = oracle.screen(obs[:c], st[:c], window=w,
                                      reset=None if reset is None else reset[:c])
            Lt, tail = tail_state(obs[:c], first, None if reset is None else reset[:c], 0, [], w)
            assert Lt == L1
            second, L2 = oracle.screen(obs[c:], st[c:], window=w, series_len=Lt, hist=tail,
                                       reset=None if reset is None else reset[c:])
            np.testing.assert_array_equal(np.concatenate([first, second]), full)
            assert L2 == L


def test_shard_bounds_cover_and_align():
    reset = np.zeros(1000, np.uint8)
    reset[[260, 505, 760]] = 1
    b = shard_bounds(1000, 4, reset)
    assert b[0][0] == 0 and b[-1][1] == 1000
    assert all(b[r][1] == b[r + 1][0] for r in range(3))
    assert [x[0] for x in b[1:]] == [260, 505, 760]
    assert shard_bounds(10, 4) == [(0, 2), (2, 5), (5, 8), (8, 10)]
