import os, sys, time, threading
sys.path.insert(0, os.getcwd())
import torch, pynvml
from paper_1903_01814_b200 import functional as F
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
B, Ci, Co, H, W = 256, 64, 128, 96, 96
x = torch.randn(B, H, W, Ci, device="cuda").to(torch.bfloat16)
w = (torch.randn(Co, Ci, 7, device="cuda") / (Ci * 7) ** 0.5).to(torch.bfloat16)
bb = torch.zeros(Co, device="cuda")
def run(label, iters=6000):
    for _ in range(50): F.conv2d_fwd_maxpool(x, w, bb, n=1)
    torch.cuda.synchronize()
    clks, pw = [], []
    stop = [False]
    def samp():
        while not stop[0]:
            clks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000)
            time.sleep(0.05)
    t = threading.Thread(target=samp); t.start()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): F.conv2d_fwd_maxpool(x, w, bb, n=1)
    e1.record(); torch.cuda.synchronize(); stop[0] = True; t.join()
    reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    clks.sort(); pw.sort()
    print(f"{label:28s} {e0.elapsed_time(e1) / iters * 1e3:7.1f} us  sm_mhz med {clks[len(clks)//2]}  power med {pw[len(pw)//2]:.0f} W  reasons 0x{reasons:x}", flush=True)
run(os.environ.get("LABEL", "default"))
