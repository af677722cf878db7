"""Complete config-4 solve of one seed by the numpy oracle (the reference restated):
    python tools/oracle_config4.py SEED [OUT_DIR] -> OUT_DIR/oracle_c4_SEED.json"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2506_04732_b200 import workloads as wl
from oracle import als_solver as als, tt_ops as ot
i=int(sys.argv[1])
r=wl.sweep_recipes()[i]
a,b,ex,_=wl.steady_problem(r)
cfg=als.Config(**r.solver)
x0=als.initial_guess(b.cores, cfg, np.random.default_rng(cfg.seed))
t=time.time()
x,rep=als.solve(a.cores,b.cores,x0=x0,cfg=cfg)
err=ot.tt_norm(ot.tt_add(x,ot.tt_scale(ex.cores,-1.0)))/ot.tt_norm(ex.cores)
json.dump({'res':list(map(float,rep.residual_history)),'ranks':list(map(int,rep.rank_history)),'err':float(err),'wall':time.time()-t}, open(os.path.join(sys.argv[2] if len(sys.argv) > 2 else '.', f'oracle_c4_{i}.json'),'w'))
print('done', i, rep.residual_history[-1], err, time.time()-t)
