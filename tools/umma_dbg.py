import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
dbg = torch.zeros(16384, device="cuda")
os.environ["MTK_UMMA_DEBUG"] = str(dbg.data_ptr())
from paper_2011_09463_b200 import api
ctx = api.Context(0)
G,M,N,K = 1,128,128,32
A = torch.arange(M*K, dtype=torch.float32).reshape(1,M,K) / 1024.0
B = torch.arange(K*N, dtype=torch.float32).reshape(1,K,N) / 1024.0
C = api.diag_gemm_tf32x3(ctx, A.cuda(), B.cuda(), False, True)
torch.cuda.synchronize()
ref = (A.double() @ B.double())
print("C sample", C[0,:2,:6].cpu().numpy(), "\nref", ref[0,:2,:6].numpy())
d = dbg.cpu().numpy()
print("smem A_hi first 40:", (d[:40]*1024).round(2))
print("smem A_hi row1:", (d[32:64]*1024).round(2))
print("smem B_hi first 40:", (d[8192:8232]*1024).round(2))
print("nonzero counts per plane:", [(d[i*4096:(i+1)*4096]!=0).sum() for i in range(4)])
