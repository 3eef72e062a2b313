import os, sys, socket
import torch, torch.distributed as dist, torch.multiprocessing as mp

def w(rank, world, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    t = torch.full((5,), float(rank + 1), device="cuda:0", dtype=torch.float64)
    dist.all_reduce(t)
    out = [torch.empty(3, device="cuda:0", dtype=torch.float64) for _ in range(world)]
    try:
        dist.all_gather(out, torch.full((3,), float(rank), device="cuda:0", dtype=torch.float64))
        ag = "ok"
    except Exception as e:
        ag = f"fail {e}"[:100]
    g = dist.new_group([0, 1])
    if rank < 2:
        u = torch.ones(2, device="cuda:0", dtype=torch.float64)
        dist.all_reduce(u, group=g)
    print(rank, t.tolist()[:1], ag, flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(w, args=(4, port), nprocs=4)
