# quick 2-process smoke of DeviceComm.allgather_ on one GPU
import os, sys, numpy as np, torch, torch.distributed as dist, torch.multiprocessing as mp
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
def w(rank, port):
    os.environ["MASTER_ADDR"]="127.0.0.1"; os.environ["MASTER_PORT"]=str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2502_16310_b200 import parallel
    torch.cuda.set_device(0)
    c = parallel.DeviceComm(1 << 20)
    for it in range(5):
        t = torch.zeros(1000, dtype=torch.int32, device="cuda")
        lo, hi = (0, 377) if rank == 0 else (377, 1000)
        t[lo:hi] = torch.arange(lo, hi, dtype=torch.int32, device="cuda") + 1000 * it
        c.allgather_(t, lo, hi)
        ok = bool((t.cpu() == torch.arange(1000, dtype=torch.int32) + 1000 * it).all())
        print(rank, it, ok, c.status(), flush=True)
    c.close()
    dist.destroy_process_group()
if __name__ == "__main__":
    import socket
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.start_processes(w, args=(port,), nprocs=2, start_method="spawn")
