import torch, time
def t(M,N,K,reps=30):
    a=torch.randn(M,K,dtype=torch.complex128,device='cuda'); b=torch.randn(N,K,dtype=torch.complex128,device='cuda')
    for _ in range(3): c=a@b.T
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): c=a@b.T
    e1.record(); e1.synchronize()
    us=e0.elapsed_time(e1)*1e3/reps
    print(M,N,K, f"{us:.1f} us {8*M*N*K/us/1e6:.2f} TF")
t(256,1024,1024); t(1024,1024,64); t(64,1024,64); t(48,128,128)
