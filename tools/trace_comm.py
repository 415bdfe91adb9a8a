"""CUPTI timeline of the sharded fused pass (GPU box helper): two ranks
(gloo for setup only) share GPU 0, each runs GridPlan.run with a DeviceComm;
rank 0 records torch.profiler traces and reports, per step, every
device->host copy and stream synchronisation with its position relative to
the level loop's exchange kernels (k_xput_marks / k_xget_marks).  The level
loop must show none between the first marking exchange and the driver's
final summary readback.

    python tools/trace_comm.py [C2] [steps]
"""

import json
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def worker(rank, port, name, steps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    import bench
    import paper_2502_16310_b200 as ow
    from paper_2502_16310_b200 import parallel, pipeline

    torch.cuda.set_device(0)
    cfg = bench.CONFIGS[name]
    data = bench.make_input(cfg)
    n = int.from_bytes(data[80:84], "little")
    rec = torch.frombuffer(bytearray(data[84:]), dtype=torch.uint8).cuda()
    comm = parallel.DeviceComm(max(64 << 20, 4 * 64 * 32 * cfg["root"] ** 3))
    plan = pipeline.GridPlan(ow.Aabb(np.zeros(3), np.ones(3)), (cfg["root"],) * 3,
                             ow.NearWallParams(d_spec=cfg["d"], n_levels=cfg["levels"], bins_per_axis=cfg["B"]),
                             cfg["lattice"], reuse_outputs=True, comm=comm)
    for _ in range(3):
        plan.run(rec, n)
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                                  torch.profiler.ProfilerActivity.CUDA])
        prof.__enter__()
    for _ in range(steps):
        if rank == 0:
            with torch.profiler.record_function("step"):
                plan.run(rec, n)
        else:
            plan.run(rec, n)
    torch.cuda.synchronize()
    if rank == 0:
        prof.__exit__(None, None, None)
        out = os.path.join("gpurun_out", f"trace_comm_{name}.json")
        prof.export_chrome_trace(out)
        report(out)
    assert comm.status() == 0
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


def report(path):
    ev = json.load(open(path))["traceEvents"]
    steps = sorted([e for e in ev if e.get("name") == "step" and e.get("ph") == "X"], key=lambda e: e["ts"])
    gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
    rt = sorted([e for e in ev if e.get("cat") == "cuda_runtime"], key=lambda e: e["ts"])
    s = steps[-1]
    t0, t1 = s["ts"], s["ts"] + s["dur"]
    ks = [k for k in gpu if t0 <= k["ts"] <= t1 + 50000]
    marks = [k for k in ks if "k_xput_marks" in k["name"] or "k_xget_marks" in k["name"]]
    d2h = [k for k in ks if k.get("cat") == "gpu_memcpy" and "DtoH" in k["name"]]
    syncs = [e for e in rt if t0 <= e["ts"] <= t1 and ("Synchronize" in e["name"] or
                                                     ("Memcpy" in e["name"] and "Async" not in e["name"]))]
    print(f"last step: wall {s['dur']:.1f} us; {len(ks)} GPU ops; exchange kernels {len(marks)}; "
          f"D2H copies {len(d2h)}; host synchronisations {len(syncs)}")
    if marks:
        lo, hi = marks[0]["ts"], marks[-1]["ts"] + marks[-1]["dur"]
        inside = [k for k in d2h if lo <= k["ts"] <= hi]
        print(f"level loop (first to last mark exchange, {hi - lo:.1f} us): {len(inside)} D2H copies")
    for k in ks:
        nm = k["name"].replace("(anonymous namespace)::", "")
        if k.get("cat") == "gpu_memcpy" or "k_x" in nm:
            print(f"  +{k['ts'] - t0:9.1f} us {k['dur']:7.1f} us  {nm[:70]}")
    for e in syncs:
        print(f"  host {e['name']} at +{e['ts'] - t0:.1f} us ({e['dur']:.1f} us)")


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mp.start_processes(worker, args=(port, name, steps), nprocs=2, start_method="spawn")
