"""Loss trajectory of the C5 training step on the bench's synthetic batches (development check)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_01814_b200.hexcnn import HexCNN  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    lr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
    import bench
    B = 256
    model = HexCNN(batch=B, lr=lr)
    xs_np, ys_np = bench.make_batches(4, B, 96, 96, 47, seed=1000)
    xs = [torch.from_numpy(a).cuda().to(torch.bfloat16) for a in xs_np]
    ys = [torch.from_numpy(a).cuda() for a in ys_np]
    out = []
    for i in range(steps):
        loss = model.step(xs[i % 4], ys[i % 4])
        out.append(float(loss.item()))
    print("lr", lr, "losses", [round(v, 4) for v in out])


if __name__ == "__main__":
    main()
