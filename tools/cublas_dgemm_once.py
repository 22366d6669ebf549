import torch
d=4096
a=torch.randn(d,d,dtype=torch.float64,device='cuda'); b=torch.randn(d,d,dtype=torch.float64,device='cuda')
for _ in range(3): c=a@b
torch.cuda.synchronize()
