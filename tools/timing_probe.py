import sys, os, torch
sys.path.insert(0, os.getcwd())
import inputs, paper_1804_05138_b200 as rq
c = inputs.CONFIGS["C2"]; m, n, k, b, p, seed = c["m"], c["n"], c["k"], c["b"], c["p"], c["seed"]
A0 = inputs.make(c["kind"], m, n, seed, device="cuda"); A = A0.t().clone().t()
ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p)
jp = torch.empty(n, dtype=torch.int64, device="cuda"); ta = torch.empty(k, dtype=torch.float64, device="cuda")
L = rq.lib()
for timing in (1, 0, 1, 0):
    L.rqrcp_set_timing(ctx._h, timing)
    for _ in range(3):
        A.copy_(A0); ctx.factor_raw(A.data_ptr(), m, m, n, k, b, p, seed, jp.data_ptr(), ta.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        A.copy_(A0); ctx.factor_raw(A.data_ptr(), m, m, n, k, b, p, seed, jp.data_ptr(), ta.data_ptr())
    e1.record(); torch.cuda.synchronize()
    print("timing", timing, "ms/step", e0.elapsed_time(e1) / 20)
