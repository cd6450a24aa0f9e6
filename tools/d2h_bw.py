import torch, time
n=8*1000*1000  # 64 MB
d=torch.zeros(n,dtype=torch.float64,device='cuda')
h=torch.empty(n,dtype=torch.float64)
hp=torch.empty(n,dtype=torch.float64).pin_memory()
torch.cuda.synchronize()
for name,dst in (('pageable',h),('pinned',hp)):
    for r in range(3):
        t=time.perf_counter(); dst.copy_(d); torch.cuda.synchronize(); dt=time.perf_counter()-t
        print(name, r, f"{dt*1e3:.1f} ms {n*8/dt/1e9:.1f} GB/s")
t=time.perf_counter(); h.copy_(hp); dt=time.perf_counter()-t; print('host memcpy 64MB', f"{dt*1e3:.1f} ms")
t=time.perf_counter(); x=torch.empty(2*n,dtype=torch.float64).pin_memory(); dt=time.perf_counter()-t; print('pin 128MB', f"{dt*1e3:.1f} ms")
import os; print('cpus', os.cpu_count())
