import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from mch_inputs import CONFIGS, make_medium
from paper_2503_01276_b200.parallel import ShardedHomogenizer
cfg = CONFIGS[2]
kap, ids = make_medium(cfg)
kd = torch.from_numpy(kap).cuda(); idd = torch.from_numpy(ids).cuda()
sh = ShardedHomogenizer(cfg, kd, idd, 0, 1)
flush = torch.empty(512*1024*1024//4, dtype=torch.float32, device="cuda")
for rep in range(4):
    sh.reset()
    if rep >= 2: flush.fill_(1.0)
    torch.cuda.synchronize()
    for l in range(1, 4):
        t0 = time.perf_counter(); sh.h.solve_level(l); t1 = time.perf_counter()
        s = sh.h.level_stats(l)
        print(rep, l, f"wall {1e3*(t1-t0):.1f} ms  ms_total {s['ms_total']:.1f} pcg {s['ms_pcg']:.1f} setup {s['ms_setup']:.1f} gram {s['ms_gram']:.1f}", flush=True)
