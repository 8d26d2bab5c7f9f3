#!/bin/bash
# One-off probe of the GPU box: topology, host RAM, CPUs, pinned H2D/D2H bandwidth.
set -x
nvidia-smi
nvidia-smi topo -m
free -g
nproc
lscpu | head -40
numactl -H 2>/dev/null || cat /sys/devices/system/node/node*/meminfo | grep MemTotal
cat /proc/meminfo | head -5
python - << 'PY'
import torch, time
d = torch.device('cuda:0')
for mb in (256, 1024, 2048):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    g = torch.empty(n, dtype=torch.uint8, device=d)
    for _ in range(3):
        g.copy_(h, non_blocking=True); h.copy_(g, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(5): g.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    h2d = 5*n/(s.elapsed_time(e)/1e3)/1e9
    s.record()
    for _ in range(5): h.copy_(g, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    d2h = 5*n/(s.elapsed_time(e)/1e3)/1e9
    # bidirectional
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); g2 = torch.empty(n, dtype=torch.uint8, device=d)
    torch.cuda.synchronize(); t0=time.time()
    for _ in range(5):
        with torch.cuda.stream(s1): g.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(g2, non_blocking=True)
    torch.cuda.synchronize(); bi = 2*5*n/(time.time()-t0)/1e9
    print(f"{mb} MB: H2D {h2d:.1f} GB/s  D2H {d2h:.1f} GB/s  bidir total {bi:.1f} GB/s")
# host memory bandwidth (numpy copy, single thread)
import numpy as np
a = np.ones(1<<28, dtype=np.float32); b = np.empty_like(a)
t0=time.time(); np.copyto(b,a); t=time.time()-t0
print("host 1-thread copy GB/s", 2*a.nbytes/t/1e9)
PY
