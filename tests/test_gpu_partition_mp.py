"""The vertex-partitioned PowerPush (BASELINE configs[4]) with two
real processes, each holding its own graph handle and part session, on the
one GPU this box has: the fused exchange stores pushed y rows through
CUDA-IPC-mapped peer buffers while the other process sweeps concurrently, the
local-phase state is broadcast from rank 0 and the sweep counters are
all-reduced over gloo. No kernel waits on another process's kernel (the
ordering is the host all-reduce between sweeps), so sharing one GPU is safe.

The assembled result is checked against the oracle's power_push: per node
|delta| <= lambda and exact r_sum <= lambda (north_star)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALPHA, LAM = 0.2, 1e-8


def _worker(rank, world, port, scale, sources, scan_threshold, fused, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2101_03652_b200 as P
        from paper_2101_03652_b200.partition import GpuPart, run_partitioned
        torch.cuda.set_device(0)
        g = P.generate_rmat(scale, 8, 11, device=0)
        n, k = g.n(), len(sources)
        part = GpuPart(g, world, rank, sources, ALPHA, LAM, scan_threshold=scan_threshold)
        res = np.zeros((k, n))
        rsd = np.zeros((k, n))
        r = run_partitioned(part, comm_device="cpu", fused=fused,
                            finish_kwargs={"reserve_ptr": res.ctypes.data,
                                           "residue_ptr": rsd.ctypes.data})
        q, cs = part.stats()
        part.close()
        t = torch.from_numpy(np.stack([res, rsd]))
        dist.all_reduce(t)  # every row is written by exactly one rank
        if rank == 0:
            np.savez(out_path, reserve=t[0].numpy(), residue=t[1].numpy(), r_sum=r.r_sum,
                     sweeps=r.sweeps, bounds=np.array(r.bounds),
                     off=g.out_offsets(), nbr=g.out_neighbors())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("fused,scan_threshold", [(True, None), (True, 40), (False, 40)])
def test_two_processes_one_gpu(oracle, tmp_path, fused, scan_threshold):
    import multiprocessing as mp
    from oracle.pyoracle import CSR
    ctx = mp.get_context("spawn")
    port = _free_port()
    out = str(tmp_path / "res.npz")
    sources = [5, 77, 1000]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 14, sources, scan_threshold, fused, out))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    d = np.load(out)
    (lo0, hi0), (lo1, hi1) = d["bounds"]
    assert lo0 == 0 and hi0 == lo1 and hi1 == len(d["off"]) - 1 and hi0 > 0
    g = CSR(d["off"], d["nbr"])
    for c, s in enumerate(sources):
        want = oracle.power_push(g, s, ALPHA, LAM, scan_threshold=scan_threshold)
        assert d["r_sum"][c] <= LAM
        assert abs(d["residue"][c].sum() - d["r_sum"][c]) <= 1e-12
        assert float(d["residue"][c].min()) >= 0.0
        assert float(np.max(np.abs(d["reserve"][c] - want.estimates))) <= LAM
