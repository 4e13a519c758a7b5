# K7 A/B (development aid): instance (rows per warp; 2 = two CTAs/SM) x T, then the phase trace
for r in 2 4; do for t in 1 2 3 4; do SOR_RES_RPW=$r python - $t <<'PY'
import os,sys,torch
sys.path.insert(0,'.')
import paper_1401_0763_b200 as P, sor_inputs as SI
T=int(sys.argv[1])
cfg=SI.config("C2"); init=torch.from_numpy(cfg.init()).cuda()
with P.Grid.create(init) as g:
    g.set_kernel("resident",T); g.iterate(cfg.omega,40); best=1e9
    for _ in range(5):
        g.reset(init); g.iterate(cfg.omega,cfg.iters); best=min(best,g.elapsed_ms)
    st=g.stats
print("rpw",os.environ["SOR_RES_RPW"],"T",T,f"{best*1e3/cfg.iters:.3f} us/iter launches {st['kernel_launches']}",flush=True)
PY
done; done
python tools/k7_trace.py
