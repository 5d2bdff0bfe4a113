import torch
a=torch.empty(28012001,dtype=torch.float64,device='cuda'); b=torch.empty_like(a)
fl=torch.empty(64*1024*1024,dtype=torch.float32,device='cuda')
for _ in range(3): a.fill_(1.0); b.fill_(2.0)
ts=[]
for i in range(10):
    fl.fill_(float(i)); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); a.fill_(1.0); b.fill_(2.0); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
print('fill 2x224MB ms', sorted(ts)[len(ts)//2])
