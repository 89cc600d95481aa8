python - << 'PY' 2>&1 | tail -45
import os, sys, time, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, '.')
os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1", MASTER_PORT="29535")
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_2403_12340_b200 import dist as D, lrgw, synth
from paper_2403_12340_b200.dist_cuda import CudaBackend
cfg = synth.CONFIGS["si64"]
psi = synth.orbitals_device(cfg, seed=1)
n_mu = lrgw.num_aux(cfg.k_mu, cfg.n_v, cfg.n_c)
def run():
    b = D.DistributedBuild(D.Comm(), CudaBackend(n_mu), cfg.dims, cfg.cell3, cfg.n_v, cfg.n_c, k_mu=cfg.k_mu, n_lambda=cfg.n_lambda, batch=128)
    b.select(psi[:, :cfg.n_v], psi[:, cfg.n_v:]); torch.cuda.synchronize()
run(); run()
import cProfile, pstats
cProfile.run('run()', '/tmp/p.prof')
p = pstats.Stats('/tmp/p.prof'); p.sort_stats('cumtime').print_stats(30)
dist.destroy_process_group()
PY
