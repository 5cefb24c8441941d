"""ResNet-18 logit error budget vs an IEEE fp32 oracle (TF32 off): python tools/resnet_err.py [batch]

Prints max |Δlogit| of the B200 forward against torchvision eager fp32 with
cuDNN/cuBLAS TF32 disabled, plus the share of each bf16 rounding source:
input image, BN-folded weights, pooled vector / fc.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    batch = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    from paper_2601_04250_b200.resnet18 import ResNet18B200, random_model
    model = random_model(0)
    x = torch.randn((batch, 3, 224, 224), generator=torch.Generator().manual_seed(1))
    m = model.cuda()
    with torch.no_grad():
        ref = m(x.cuda()).float()
        ref_xb = m(x.cuda().bfloat16().float()).float()
    net = ResNet18B200(model, max_batch=batch)
    out = net.forward(x.cuda()).clone()
    torch.cuda.synchronize()
    s = 7
    last = net.stage_bufs[3][1]
    fm = last[(s + 2) * 512:].view(-1, 512)[: batch * (s + 1) * (s + 1)].view(batch, s + 1, s + 1, 512)
    pooled32 = fm[:, :s, :s].float().mean(dim=(1, 2))
    fc32 = torch.nn.functional.linear(pooled32, m.fc.weight.float(), m.fc.bias.float())
    fc_bfpool = torch.nn.functional.linear(net.pooled[:batch].float(), m.fc.weight.float(), m.fc.bias.float())
    del fm

    def e(a):
        return (a - ref).abs().max().item()
    print(f"batch {batch}: logit scale {ref.abs().max().item():.3f}")
    print(f"  ours (fp16 convs, fp32 head)    max|d| = {e(out):.4e}  argmax agree "
          f"{(out.argmax(1) == ref.argmax(1)).float().mean().item():.4f}")
    print(f"  ours map + torch fp32 pool/fc   max|d| = {e(fc32):.4e}")
    print(f"  ours pooled + torch fp32 fc     max|d| = {e(fc_bfpool):.4e}")
    print(f"  fp32 model on bf16-rounded input max|d| = {e(ref_xb):.4e}")
    with torch.no_grad():
        torch.backends.cudnn.allow_tf32 = True
        ref_tf32 = m(x.cuda()).float()
    print(f"  TF32 oracle vs IEEE oracle      max|d| = {e(ref_tf32):.4e}")


if __name__ == "__main__":
    main()
