import torch, time
torch.cuda.init()
d = torch.device("cuda")
for n in (64, 65536, 1<<20, 1<<22, 1<<25):
    xs=[]
    torch.cuda.synchronize()
    t0=time.perf_counter()
    for i in range(2000):
        x = torch.empty(n, dtype=torch.float64, device=d)
        xs.append(x)
        if len(xs) > 20: xs.pop(0)
    t1=time.perf_counter()
    print(n, (t1-t0)/2000*1e6, "us per torch.empty")
import ctypes
t0=time.perf_counter()
for i in range(2000):
    b = torch.empty(96, dtype=torch.uint8, device=d)
t1=time.perf_counter(); print("uint8 96B", (t1-t0)/2000*1e6)
