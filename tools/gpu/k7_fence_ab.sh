# K7 release variants on C2 (development aid)
for i in 1 2; do for lib in libsor.so libsor_relaxpoll.so; do
SOR_LIBRARY=paper_1401_0763_b200/$lib python - <<'PY'
import os,sys,torch
sys.path.insert(0,'.')
import paper_1401_0763_b200 as P, sor_inputs as SI
cfg=SI.config("C2"); init=torch.from_numpy(cfg.init()).cuda()
with P.Grid.create(init) as g:
    g.set_kernel("resident",3); g.iterate(cfg.omega,40); best=1e9
    for _ in range(5):
        g.reset(init); g.iterate(cfg.omega,cfg.iters); best=min(best,g.elapsed_ms)
print(os.path.basename(os.environ["SOR_LIBRARY"]), f"C2 T=3 {best*1e3/cfg.iters:.3f} us/iter", flush=True)
PY
done; done
