"""Peer-copy bandwidth through the fabric (one process per GPU, torchrun).

Every rank allocates a buffer in its device heap; rank r then times
rdmm_memcpy (cudaMemcpyAsync, copy engine) from rank (r+d) % P's heap into a
local buffer, for each distance d, with all ranks copying at once.  Prints
one JSON line per (size, distance) from rank 0 with the max-over-ranks time.
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch
import torch.distributed as dist

import paper_2311_18141_b200.dist as dm
from paper_2311_18141_b200 import _lib as L


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    obj = [f"p2p{os.getpid()}" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    sizes = [64 << 20, 256 << 20]
    heap = 2 * max(sizes) + (64 << 20)
    f = dm.Fabric(nranks=world, heap_bytes=heap, first_local=rank, nlocal=1,
                  devices=[rank], session=obj[0])
    h = f.handle
    src = L.Gptr()
    dst = L.Gptr()
    L.check(L.rdmm_heap_alloc(h, rank, max(sizes), C.byref(src)))
    L.check(L.rdmm_heap_alloc(h, rank, max(sizes), C.byref(dst)))
    offs = [None] * world
    dist.all_gather_object(offs, src.offset)
    dptr = C.c_void_p()
    L.check(L.rdmm_gptr_device(h, rank, dst, C.byref(dptr)))
    L.check(L.rdmm_memset(dptr, 1, max(sizes), None))
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    for nb in sizes:
        for d in range(1, world):
            peer = (rank + d) % world
            g = L.Gptr(peer, 0, offs[peer], nb)
            pp = C.c_void_p()
            L.check(L.rdmm_gptr_device(h, rank, g, C.byref(pp)))
            reps = 5
            times = []
            for it in range(reps + 2):
                dist.barrier()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    e0.record(s)
                    L.check(L.rdmm_memcpy(dptr, pp, nb, C.c_void_p(s.cuda_stream)))
                    e1.record(s)
                s.synchronize()
                if it >= 2:
                    times.append(e0.elapsed_time(e1))
            t = torch.tensor([min(times), sum(times) / len(times)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(json.dumps({"bytes": nb, "distance": d, "world": world,
                                  "ms_min": t[0].item(), "ms_avg": t[1].item(),
                                  "GBps_per_rank": nb / t[0].item() / 1e6}), flush=True)
    dist.barrier()
    f.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
