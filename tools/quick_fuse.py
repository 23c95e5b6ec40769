import sys, time, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2601_03067_b200 import _native as N
from paper_2601_03067_b200.engine import FusionEngine, Geometry
from paper_2601_03067_b200.schedule import bff_plan
from paper_2601_03067_b200.workload import synthetic_kv
L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B, p, t, h, d = 64, 256, 16, 8, 128
t0 = time.time()
Kt, Vt = synthetic_kv(L, B, p, t, h, d, dtype=torch.bfloat16, seed=1)
torch.cuda.synchronize(); print('gen', time.time() - t0, flush=True)
geom = Geometry(L, B * p, t, h, d, 0); plan = bff_plan(B, p, None)
for path in (N.PATH_TC,):
    eng = FusionEngine(geom, plan, torch.bfloat16, Kt.device, path)
    for it in range(3):
        k, v = Kt.clone().reshape(-1), Vt.clone().reshape(-1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); st = eng.run(k, v, 0.8, time_sim=True); e1.record(); torch.cuda.synchronize()
        tot = e0.elapsed_time(e1)
        sims = [(a.elapsed_time(b)) for a, b, _ in st.sim_events]
        flops = 0.0
        for lv_stats in st.level_stats:
            s = lv_stats.cpu().double()
            flops += float((2 * s[..., 0] * s[..., 1] * geom.r).sum())
        nb = st.live_count.sum().item()
        print(f'path {path} total {tot:.2f} ms sim {sum(sims):.2f} ms {[round(x,2) for x in sims]} '
              f'alg TFLOP/s {flops/sum(sims)/1e9:.1f} CR {L*B*p/nb:.4f} KV GB/s {2*L*B*p*t*h*d*2/tot/1e6:.1f}', flush=True)
