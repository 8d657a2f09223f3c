import torch, time
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
f = torch.empty(64*1024*1024, dtype=torch.float32, device="cuda")
for _ in range(3): f.zero_()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(12)]
for i in range(6):
    ev[2*i].record(s); f.zero_(); ev[2*i+1].record(s)
torch.cuda.synchronize()
print("zero_ ms", [round(ev[2*i].elapsed_time(ev[2*i+1]),3) for i in range(6)])
x = torch.empty(64*1024*1024, dtype=torch.float32, device="cuda")
for i in range(6):
    ev[2*i].record(s); x.copy_(f); ev[2*i+1].record(s)
torch.cuda.synchronize()
print("copy ms", [round(ev[2*i].elapsed_time(ev[2*i+1]),3) for i in range(6)])
