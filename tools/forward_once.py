"""One warm forward (for ncu launch lists / captures): python tools/forward_once.py resnet18|distilbert [reps]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    if which == "resnet18":
        from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
        net = ResNet18B200(random_model(0), max_batch=64)
        x = torch.randn((64, 3, 224, 224), device="cuda")
        for _ in range(reps):
            net.forward(x)
    else:
        from paper_2601_04250_b200.distilbert import DistilBertB200, random_model
        net = DistilBertB200(random_model(0), max_batch=128)
        ids = torch.randint(0, 30522, (128, 128), device="cuda", dtype=torch.int32)
        for _ in range(reps):
            net.forward(ids)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
