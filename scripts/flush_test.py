import torch, time
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
for mb in (64, 256, 512):
    f = torch.empty(mb * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    f.zero_(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10): f.zero_()
    e1.record(s); torch.cuda.synchronize()
    print(mb, "MB zero_ x10:", e0.elapsed_time(e1), "ms")
    e0.record(s)
    for i in range(10): f.fill_(float(i))
    e1.record(s); torch.cuda.synchronize()
    print(mb, "MB fill_ x10:", e0.elapsed_time(e1), "ms")
