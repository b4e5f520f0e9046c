"""One process per rank (the torchrun layout) on the GPU: two processes
share the fabric by session name (CUDA-IPC-mapped heaps, shared-memory
control segment) and run every variant of run_multiply, compared with the
oracle.  Both ranks may sit on the same GPU (IPC works within a device), so
this runs on a one-GPU box; with two GPUs each process gets its own."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
VARIANTS = ["summa_bsp", "stationary_c", "stationary_a", "stationary_b", "ws_random",
            "ws_locality"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2311_18141_b200.dist as dm

    orc = oracle.port()
    name = [f"mp{os.getpid()}_{port}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    res = {}
    f = dm.Fabric(nranks=world, heap_bytes=64 << 20, first_local=rank, nlocal=1, devices=[dev],
                  session=name[0])
    g = dm.ProcGrid(1, 2)
    m, k, n = 40, 36, 24
    ga = orc.random_csr(m, k, 0.3, 11, dtype=np.float64)
    gb = orc.random_dense(k, n, 12, dtype=np.float64)
    want = np.zeros((m, n))
    orc.spmm_local(ga, gb, want)
    gs = orc.random_csr(k, n, 0.3, 13, dtype=np.float64)
    sw, _ = orc.spgemm_local(ga, gs)
    for v in VARIANTS[1:]:
        A = dm.DistSparse(f, m, k, 20, 9, g, 0, dtype=np.float64)
        B = dm.DistDense(f, k, n, 9, 6, g, 1, dtype=np.float64)
        C = dm.DistDense(f, m, n, 20, 6, g, 2, dtype=np.float64)
        A.init_from_global(ga.row_ptr, ga.col_idx, ga.values)
        B.init_from_global(gb)
        C.init()
        rep = dm.run_multiply(f, A, B, C, variant=v, record_triples=True)
        res[("spmm", v)] = bool(np.array_equal(C.to_global(), want))
        res[("triples", v)] = len(rep.triples)
        Bs = dm.DistSparse(f, k, n, 9, 6, g, 1, dtype=np.float64)
        Cs = dm.DistSparse(f, m, n, 20, 6, g, 2, dtype=np.float64)
        Bs.init_from_global(gs.row_ptr, gs.col_idx, gs.values)
        Cs.init()
        dm.run_multiply(f, A, Bs, Cs, variant=v)
        rp, ci, vv = Cs.to_global()
        res[("spgemm", v)] = bool(np.array_equal(rp, sw.row_ptr) and np.array_equal(ci, sw.col_idx)
                                  and np.array_equal(vv, sw.values))
        for mat in (A, B, C, Bs, Cs):
            mat.close()
    f.close()
    out[rank] = res
    dist.destroy_process_group()


def test_two_processes_every_variant():
    port = _port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    for rank in (0, 1):
        for v in VARIANTS[1:]:
            assert out[rank][("spmm", v)], (rank, v)
            assert out[rank][("spgemm", v)], (rank, v)
    # each process records its own rank's triples; together they cover M*N*K
    for v in VARIANTS[1:]:
        assert out[0][("triples", v)] + out[1][("triples", v)] == 2 * 4 * 4
