import torch, time
n = 268435456 // 4
for pinned in (True,):
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device='cuda')
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print('h2d GB/s', 5*n*4/e0.elapsed_time(e1)/1e6)
    e0.record(); 
    for _ in range(5): h.copy_(d, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print('d2h GB/s', 5*n*4/e0.elapsed_time(e1)/1e6)
    # chunked 8
    c = n // 8
    s = torch.cuda.Stream()
    e0.record(s)
    with torch.cuda.stream(s):
        for k in range(8): d[k*c:(k+1)*c].copy_(h[k*c:(k+1)*c], non_blocking=True)
    e1.record(s); torch.cuda.synchronize()
    print('h2d chunked GB/s', n*4/e0.elapsed_time(e1)/1e6)
