"""T4 on the GPU: the data-parallel product path with two ranks.

Two processes share cuda:0 (the test box has one GPU; NCCL refuses two ranks on
one device, so the process group is gloo, which all-reduces CUDA tensors).  Each
rank takes its LPT shard of a variable-length utterance pool (P:364-368,
length-bucketed batches), runs lfmmi_loss_grad through the C-ABI on it and
all-reduces the 5 float64 totals with paper_2112_00709_b200.dist.  The reduced
totals must equal a one-rank run over the whole pool to 1e-12 relative (the
utterances are independent, only the summation order differs) and the oracle
within the gates; every rank's gradient rows equal the one-rank rows bit for bit
(per-utterance outputs do not depend on batch composition, §8(b))."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2112_00709_b200 import dist as fdist
from paper_2112_00709_b200 import synth

pytestmark = pytest.mark.gpu

N_POOL, D = 24, 500


def _pool():
    lens, nums, den = synth.make_c5_utterances(seed=5, B=N_POOL, K=1500, nnz=10000, D=D)
    lens = np.minimum(lens, 120).astype(np.int32)
    nums = [synth.numerator_graph(np.random.Generator(np.random.PCG64(100 + i)), int(max(5, n // 3)), D, "random")
            for i, n in enumerate(lens.tolist())]
    emis = synth.c5_emissions(5, np.arange(N_POOL), int(lens.max()), D)
    return lens, nums, den, emis


def _shards(world):
    lens, nums, den, _ = _pool()
    costs = fdist.utterance_costs(lens, [g.nnz for g in nums], den.nnz)
    return fdist.lpt_shard(costs, world)


def _run(idx):
    """lfmmi_loss_grad on utterances idx of the pool, on cuda:0; returns device tensors."""
    import torch

    import paper_2112_00709_b200 as fbx

    lens, nums, den, emis = _pool()
    n_max = int(lens[idx].max())
    e = torch.from_numpy(np.ascontiguousarray(emis[idx][:, :n_max])).cuda()
    L = torch.from_numpy(lens[idx]).cuda()
    num_g = fbx.Graph.from_host(synth.compose([nums[i] for i in idx]))
    den_g = fbx.Graph.from_host(den)
    loss, totals, st, grad = fbx.lfmmi_loss_grad(num_g, den_g, e, L)
    torch.cuda.synchronize()
    return loss, totals, st, grad


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        idx = _shards(world)[rank]
        loss, totals, st, grad = _run(idx)
        fdist.allreduce_totals(totals)  # gloo all-reduce of a CUDA tensor
        torch.cuda.synchronize()
        q.put((rank, idx.tolist(), totals.cpu().numpy().tolist(), loss.cpu().numpy(), st.cpu().numpy(),
               grad.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_share_one_gpu_product_path():
    import torch

    assert torch.cuda.is_available()
    from paper_2112_00709_b200 import build

    build.build()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    got.sort(key=lambda x: x[0])
    # both ranks hold the same reduced totals
    assert got[0][2] == got[1][2]
    assert sorted(got[0][1] + got[1][1]) == list(range(N_POOL))
    # one rank over the whole pool (longest-first order, as the sharder would give it)
    all_idx = _shards(1)[0]
    loss1, tot1, st1, grad1 = _run(all_idx)
    tot1 = tot1.cpu().numpy()
    red = np.array(got[0][2])
    assert red[1] == tot1[1] and red[4] == tot1[4] == 0
    for i in (0, 2, 3):
        assert abs(red[i] - tot1[i]) <= 1e-12 * abs(tot1[i]), (i, red[i], tot1[i])
    # per-utterance outputs are bitwise independent of the shard they ran in
    pos = {u: k for k, u in enumerate(all_idx.tolist())}
    loss1, grad1 = loss1.cpu().numpy(), grad1.cpu().numpy()
    for _, idx, _, loss, st, grad in got:
        assert (st == 0).all()
        for k, u in enumerate(idx):
            assert loss[k] == loss1[pos[u]]
            n = grad.shape[1]
            assert (grad[k] == grad1[pos[u], :n]).all() and (grad1[pos[u], n:] == 0).all()
    # and the oracle's totals within the gates
    lens, nums, den, emis = _pool()
    ref = oracle.lfmmi_batch(synth.compose(nums), synth.compose([den]), emis, lens)["totals"]
    assert red[1] == ref[1] and red[4] == ref[4]
    for i in (0, 2, 3):
        assert abs(red[i] - ref[i]) <= 1e-5 * max(1.0, abs(ref[3])), (i, red[i], ref[i])
