"""A few 3-D fused iterations at 512^3 (development aid: ncu target)."""
import sys
sys.path.insert(0, ".")
import paper_1401_0763_b200 as P  # noqa: E402
import sor_inputs as SI  # noqa: E402
dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
init = SI.random_shell3d(512, 512, 512, seed=7)
with P.Grid3D(init, dtype=dtype) as g:
    g.set_kernel("fused")
    g.iterate(1.9, 3)
