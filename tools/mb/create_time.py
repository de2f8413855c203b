"""Development aid: device time of ils_create on a config, repeated, optionally with an SP solve
and an L2 flush in between (the bench's step pattern)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2203_15340_b200 import ils
from workloads import make_problem
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "plain"
pr = make_problem(cfg)
A = torch.from_numpy(pr.A).cuda(); b = torch.from_numpy(pr.b).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
for i in range(6):
    if mode != "plain":
        flush.fill_(float(i))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    h = ils.ils_create(A, b, pr.p, pr.q, pr.n, stream=torch.cuda.current_stream().cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if mode == "solve":
        ils.ils_sp_solve(h, None, x, 0.0, 2, ils.ils_default_opts(stop=ils.ILS_STOP_NONE))
    ils.ils_destroy(h)
    torch.cuda.synchronize()
    print(f"{cfg} {mode}: create device {e0.elapsed_time(e1):.2f} ms wall {1e3 * (t1 - t0):.2f} ms", flush=True)
