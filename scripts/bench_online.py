"""Online instrumentation slowdowns (instrumented / plain kernel time), C1, C3, C4."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_04701_b200 import hirace as hr, online as on
from tracegen import c4

out = {}
d1 = torch.arange(8 * 256 + 8, dtype=torch.int32, device="cuda")
ck = hr.Checker(8 * 256 + 8, 256)
out["c1"] = on.slowdown(lambda: on.c1(None, d1, False), lambda: on.c1(ck.ctx, d1, True), reps=20)
ck.close()
d3 = torch.randint(0, 100, (2 * 512 * 512,), dtype=torch.int32, device="cuda")
ck = hr.Checker(2 * 512 * 512, 648)
out["c3"] = on.slowdown(lambda: on.c3(None, d3, False), lambda: on.c3(ck.ctx, d3, True), reps=10)
ck.close()
lv = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = c4.Graph(lv)
dev = on.C4Device(g)
d4 = torch.zeros(g.n + 1024, dtype=torch.int32, device="cuda")
ck = hr.Checker(g.n + 1024, 0, ring_capacity=1 << 24)
for racy in (False, True):
    out[f"c4_{'racy' if racy else 'atomic'}"] = on.slowdown(lambda: dev.run(None, d4, False, racy),
                                                            lambda: dev.run(ck.ctx, d4, True, racy), reps=5)
ck.close()
print(json.dumps({k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in out.items()}))
