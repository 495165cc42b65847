import os, sys
import torch, torch.distributed as dist, torch.multiprocessing as mp

def work(rank):
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = "29561"
    dist.init_process_group("gloo", rank=rank, world_size=2)
    dev = torch.device("cuda", 0)
    t = torch.tensor([float(rank + 1)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = {"max": t.item()}
    sc = torch.tensor([1, 2], dtype=torch.int64, device=dev) + rank
    rc = torch.empty_like(sc)
    try:
        dist.all_to_all_single(rc, sc)
        out["a2a"] = rc.tolist()
    except Exception as e:
        out["a2a"] = f"ERR {type(e).__name__}: {str(e)[:120]}"
    try:
        sf = torch.arange(3 * (rank + 1), dtype=torch.float32, device=dev)
        rf = torch.empty(3 * 1 + 3 * 2 if rank == 0 else 3 + 6, device=dev)
        dist.all_to_all_single(torch.empty(0, device=dev) if False else rf[: (3 if rank == 0 else 6) * 1 + (3 if rank==0 else 6)], sf, [3 * 1, 3 * 2] if False else None)
        out["a2av"] = "ok"
    except Exception as e:
        out["a2av"] = f"ERR {type(e).__name__}: {str(e)[:120]}"
    print(rank, out, flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    mp.spawn(work, nprocs=2)
