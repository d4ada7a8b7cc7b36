for shape in "256 64 128 96 96 1" "256 128 128 48 48 2" "256 256 256 24 24 2"; do
for m in 0 1 2; do
HEXCONV_WG_DEBUG=$m python - <<PY
import torch, sys
sys.path.insert(0,'.')
from paper_1903_01814_b200 import functional as F
B,Ci,Co,H,W,n = map(int, "$shape".split())
T=F.num_taps(n)
x=torch.randn(B,H,W,Ci,device='cuda').to(torch.bfloat16); g=torch.randn(B,H,W,Co,device='cuda').to(torch.bfloat16)
for _ in range(3): F.conv2d_bwd_weight(x,g,n=n,layout='NHWC')
torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5): F.conv2d_bwd_weight(x,g,n=n,layout='NHWC')
e.record(); torch.cuda.synchronize()
print("$shape", "dbg=$m", round(s.elapsed_time(e)/5*1000,1), "us")
PY
done; done
