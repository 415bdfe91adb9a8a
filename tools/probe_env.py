import os, time, torch
print({k: v for k, v in os.environ.items() if "TORCH" in k or "CUDA" in k})
print("backend", torch.cuda.get_allocator_backend())
x = torch.empty(10, device="cuda")
for sync in (False, True):
    ts = []
    for it in range(20):
        t0 = time.perf_counter()
        y = [torch.empty(250000, dtype=torch.int32, device="cuda") for _ in range(7)]
        if sync:
            torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del y
    print("sync" if sync else "nosync", [round(1e3 * t, 3) for t in ts])
print(torch.cuda.memory_stats()["num_alloc_retries"], torch.cuda.memory_stats()["segment.all.allocated"])
