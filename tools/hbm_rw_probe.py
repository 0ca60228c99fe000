"""HBM bandwidth by direction with torch kernels over a 17.2 GB f32 tensor (the configs[4]
input / output size): pure read (sum), copy, pure write (fill).  One B200, round 2:
read 6.51 TB/s, copy 6.67 TB/s (read + write bytes), write 7.51 TB/s."""
import torch, time
dev=torch.device('cuda',0)
a=torch.empty((1<<20, 4096), dtype=torch.float32, device=dev).normal_()
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    ts=[]
    for _ in range(n):
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
ms=t(lambda: a.sum())
print('sum read   %.3f ms  %.2f TB/s' % (ms, a.numel()*4/ms/1e9))
ms=t(lambda: a.view(-1)[:1<<31].max())
print('max read 8GB %.3f ms  %.2f TB/s' % (ms, (1<<31)*4/ms/1e9))
b=torch.empty_like(a)
ms=t(lambda: b.copy_(a))
print('copy       %.3f ms  %.2f TB/s (r+w)' % (ms, 2*a.numel()*4/ms/1e9))
ms=t(lambda: b.fill_(1.0))
print('fill write %.3f ms  %.2f TB/s' % (ms, a.numel()*4/ms/1e9))
