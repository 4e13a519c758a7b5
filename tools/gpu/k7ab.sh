# K7 A/B (development aid): rows per warp (2: two CTAs/SM) x T on C2
for r in ${RPWS:-2 4}; do for t in ${TS:-1 2 3 4}; do SOR_RES_RPW=$r SOR_RESIDENT_T=$t python - <<'PY'
import os,sys,torch
sys.path.insert(0,'.')
import paper_1401_0763_b200 as P, sor_inputs as SI
cfg=SI.config("C2"); init=torch.from_numpy(cfg.init()).cuda()
with P.Grid.create(init) as g:
    g.set_kernel("resident",3); g.iterate(cfg.omega,40); best=1e9
    for _ in range(5):
        g.reset(init); g.iterate(cfg.omega,cfg.iters); best=min(best,g.elapsed_ms)
    st=g.stats
print("rpw",os.environ["SOR_RES_RPW"],"T",os.environ["SOR_RESIDENT_T"],f"{best*1e3/cfg.iters:.3f} us/iter launches {st['kernel_launches']}",flush=True)
PY
done; done
