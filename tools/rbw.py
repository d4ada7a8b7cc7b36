import torch
x = torch.empty(2**30, dtype=torch.bfloat16, device="cuda").normal_()
y = torch.empty_like(x)
def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
ms = t(lambda: x.amax()); print("read-only amax  %.1f GB/s" % (2**31 / ms / 1e6))
ms = t(lambda: x.sum(dtype=torch.float32)); print("read-only sum   %.1f GB/s" % (2**31 / ms / 1e6))
ms = t(lambda: y.copy_(x)); print("copy            %.1f GB/s" % (2**32 / ms / 1e6))
ms = t(lambda: y.fill_(1.0)); print("write-only fill %.1f GB/s" % (2**31 / ms / 1e6))
