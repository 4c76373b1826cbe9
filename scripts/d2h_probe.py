import sys, time, os
sys.path.insert(0, '/root/repo')
import torch
from paper_1711_03888_b200 import hostio
n = 6 * 262144000
src = torch.empty(n, dtype=torch.float32, device='cuda').fill_(1.0)
print("threads", torch.get_num_threads(), os.cpu_count())
for chunk in (64 << 20, 256 << 20):
    hostio.CHUNK = chunk
    for rep in range(3):
        host = hostio.empty_host(n)
        torch.cuda.synchronize(); t = time.perf_counter()
        hostio.to_host(src.view(torch.uint8), host.view(torch.uint8))
        dt = time.perf_counter() - t
        print(f"chunk {chunk>>20} MB: {dt*1e3:.0f} ms {4*n/dt/1e9:.1f} GB/s", flush=True)
pin = torch.empty(n, dtype=torch.float32, pin_memory=True)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    pin.copy_(src); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"pinned DMA only: {dt*1e3:.0f} ms {4*n/dt/1e9:.1f} GB/s")
for rep in range(2):
    host = hostio.empty_host(n)
    t = time.perf_counter(); host.copy_(pin); dt = time.perf_counter() - t
    print(f"cpu copy pinned->fresh: {dt*1e3:.0f} ms {4*n/dt/1e9:.1f} GB/s")
host = hostio.empty_host(n); host.fill_(0)
t = time.perf_counter(); host.copy_(pin); dt = time.perf_counter() - t
print(f"cpu copy pinned->touched: {dt*1e3:.0f} ms {4*n/dt/1e9:.1f} GB/s")
