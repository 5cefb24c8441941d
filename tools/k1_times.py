import sys, os
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2601_04250_b200 as gg
from paper_2601_04250_b200 import _abi
n = 1 << 26
c = torch.rand(n, device="cuda", dtype=torch.float64) * 0.5 + 0.5
scores = torch.stack([c, 1.0 - c], dim=1).contiguous()
now = torch.linspace(0.0, 10.0, n, device="cuda", dtype=torch.float64)
ctl = gg.ControllerConfig(alpha=1.0, beta=-0.1, gamma=-0.3, tau0=0.9, tau_inf=0.4, k=0.5,
                          routing=gg.RoutePolicy.THRESHOLD_ON_QUEUE).build(gg.EnergyLedger())
snap = torch.frombuffer(bytearray(bytes(_abi.gg_snapshot(3, 7.5, 0.25))), dtype=torch.uint8).cuda()
out = ctl.decide_batch(scores, now, snap, breakdown=False)
for _ in range(3): ctl.decide_batch(scores, now, snap, breakdown=False, out=out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5): ctl.decide_batch(scores, now, snap, breakdown=False, out=out)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
from collections import defaultdict
agg = defaultdict(list)
for e in evs: agg[e.name[:70]].append(e.device_time if hasattr(e,'device_time') else e.cuda_time)
for k, v in agg.items(): print(f"{sum(v)/len(v):9.1f} us x{len(v)}  {k}")
