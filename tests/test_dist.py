"""T4: data-parallel logic on CPU (gloo, world size 2).

The sharding covers every utterance exactly once and balances cost; per-rank
totals all-reduced over gloo equal the single-process totals of the whole pool
(computed with the oracle, since this container has no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2112_00709_b200 import dist as fdist
from paper_2112_00709_b200 import synth


def test_lpt_covers_once_and_balances():
    rng = np.random.default_rng(0)
    costs = rng.lognormal(5, 0.5, 1024)
    for world in (1, 2, 4, 8):
        shards = fdist.lpt_shard(costs, world)
        allidx = np.concatenate(shards)
        assert sorted(allidx.tolist()) == list(range(1024))
        loads = [costs[s].sum() for s in shards]
        assert max(loads) - min(loads) <= costs.max() + 1e-9
        for s in shards:
            assert (np.diff(costs[s]) <= 0).all()  # longest first within a rank


def _pool():
    lens, nums, den = synth.make_c5_utterances(seed=5, B=12, K=300, nnz=1500, D=200)
    lens = np.minimum(lens, 60).astype(np.int32)
    nums = [synth.numerator_graph(np.random.Generator(np.random.PCG64(i)), int(max(5, n // 3)), 200, "random")
            for i, n in enumerate(lens.tolist())]
    emis = synth.c5_emissions(5, np.arange(12), 60, 200)
    return lens, nums, den, emis


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lens, nums, den, emis = _pool()
    costs = fdist.utterance_costs(lens, [g.nnz for g in nums], den.nnz)
    idx = fdist.lpt_shard(costs, world)[rank]
    r = oracle.lfmmi_batch(synth.compose([nums[i] for i in idx]), synth.compose([den]), emis[idx], lens[idx])
    t = torch.tensor(r["totals"], dtype=torch.float64)
    fdist.allreduce_totals(t)
    if rank == 0:
        q.put(t.numpy().tolist())
    dist.destroy_process_group()


def test_gloo_allreduce_equals_single_process():
    import oracle

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    lens, nums, den, emis = _pool()
    ref = oracle.lfmmi_batch(synth.compose(nums), synth.compose([den]), emis, lens)["totals"]
    assert got[1] == ref[1] and got[4] == ref[4]
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-9)
