"""The sharded data path (paper_2410_06074_b200.dist.sharded_step) with two
processes on one GPU (gloo carries the collectives through host memory; the
round's GPU box has a single B200): the gathered y, the reduced loss and every rank's shard of the
gradients must equal the single-process call bit for bit -- instances are
independent, so a shard's kernels compute exactly what the full batch's do."""

import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2410_06074_b200 as smnn
        from paper_2410_06074_b200 import dist as sd
        from synth.workloads import make_grad_y, make_workload_inputs, workload

        torch.cuda.set_device(0)
        wl = workload("sst").with_(D=101)  # 101 instances: uneven shards
        x = make_workload_inputs(wl, seed=3)
        gy = torch.from_numpy(make_grad_y(wl.n_inst, wl.T, wl.order, dtype="f32", seed=4))
        full = {k: torch.from_numpy(v).cuda() for k, v in x.items()}
        for compute in ("f64", None):
            y_all, loss, g = sd.sharded_step(smnn, full, gy.cuda(), rank, world, compute=compute)
            torch.cuda.synchronize()
            assert int(g[4].abs().max()) == 0
            q.put((rank, compute, y_all.cpu().numpy(), float(loss), [t.cpu().numpy() for t in g[:4]]))
    finally:
        dist.destroy_process_group()


def test_sharded_step_matches_single_process():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2410_06074_b200 as smnn
    from paper_2410_06074_b200 import dist as sd
    from synth.workloads import make_grad_y, make_workload_inputs, workload

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, 29631, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(4)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    wl = workload("sst").with_(D=101)
    x = make_workload_inputs(wl, seed=3)
    gy = torch.from_numpy(make_grad_y(wl.n_inst, wl.T, wl.order, dtype="f32", seed=4)).cuda()
    t = {k: torch.from_numpy(v).cuda() for k, v in x.items()}
    for compute in ("f64", None):
        # the same calls sharded_step makes (f32c64: the y_lo hand-off where the pipeline takes it)
        lo = compute == "f64" and smnn.ylo_used(t["coeffs"], t["iv"], compute=compute)
        out = smnn.smnn_factor_solve_fwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], compute=compute, with_ylo=lo)
        y = out[0]
        g = smnn.smnn_solve_bwd(t["coeffs"], t["rhs"], t["iv"], t["steps"], y, gy, compute=compute,
                                y_lo=out[2] if lo else None)
        loss = float((gy.double() * y.double()).sum())
        mine = [r for r in res if r[1] == compute]
        assert len(mine) == 2
        for rank, _, y_all, l, gl in mine:
            assert np.array_equal(y_all, y.cpu().numpy())
            assert abs(l - loss) <= 1e-12 * abs(loss)
            s, e = sd.shard_range(wl.n_inst, rank, 2)
            for a, b in zip(gl, g[:4]):
                assert np.array_equal(a, b[s:e].cpu().numpy())
