"""World-size-2 test of the sharded trainer's host logic on CPU (gloo):
consecutive-block window assignment (sharding.rank_windows / plan) plus the
per-batch gradient all-reduce of sharding.run_sharded_epoch, with a session
double whose per-window gradients come from the compiled reference. The
all-reduced, 1/W-scaled gradient must equal the reference's distributed
epoch gradient (src/distsim.cpp:248-260)."""
import os
import socket

import numpy as np
import pytest

N, DEG, DIM, T = 80, 3, 4, 9
L_, S_, H_ = 3, 1, 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class RefWindowSession:
    """Test double of the C-ABI session: local_grads = sum of reference
    per-window gradients over this rank's consecutive window block."""

    def __init__(self, rank, world):
        from oracle import refbind as R
        from paper_2501_15348_b200.sharding import rank_windows
        self.g = R.RefGraph.synth(N, DEG, DIM, T, 0.1, 0.05, seed=3)
        self.cfg = R.RunCfg(arch="tgcn", hidden=8, seq_len=L_, horizon=H_)
        self.W = len(R.sliding_windows(T - 1, L_, S_, H_))
        self.wb, self.we = rank_windows(T - 1, world, rank, L_, S_, H_)
        self.applied = None

    def begin_epoch(self):
        return 1

    def local_grads(self, b, grad):
        import torch
        acc = np.zeros(grad.numel())
        for w in range(self.wb, self.we):
            acc += self.g.sample_grads(self.cfg, w)[2]
        grad.copy_(torch.from_numpy(acc))

    def apply(self, grad):
        self.applied = grad.numpy() / self.W
        return True

    def end_epoch(self):
        pass


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2501_15348_b200.sharding import run_sharded_epoch, torch_allreduce
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = RefWindowSession(rank, world)
        grad = torch.zeros(s.g.num_params(s.cfg), dtype=torch.float64)
        flags = run_sharded_epoch(s, grad, torch_allreduce(world))
        q.put((rank, s.wb, s.we, flags, s.applied))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_allreduce_matches_reference_distributed_gradient(ref):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # consecutive blocks partition all windows, counts differ by <= 1
    W = len(ref.sliding_windows(T - 1, L_, S_, H_))
    blocks = [(r[1], r[2]) for r in res]
    assert blocks[0][0] == 0 and blocks[-1][1] == W and blocks[0][1] == blocks[1][0]
    assert abs((blocks[0][1] - blocks[0][0]) - (blocks[1][1] - blocks[1][0])) <= 1
    # every rank applies the identical all-reduced step
    assert all(r[3] == [True] for r in res)
    assert np.array_equal(res[0][4], res[1][4])
    g = ref.RefGraph.synth(N, DEG, DIM, T, 0.1, 0.05, seed=3)
    want = g.run(ref.RunCfg(arch="tgcn", hidden=8, seq_len=L_, horizon=H_, workers=2)).grads0
    assert np.allclose(res[0][4], want, rtol=1e-9, atol=1e-12)
