"""K7 per-pass timeline (development aid): run C2 with SOR_RES_TRACE and
summarise each pass (globaltimer ns, thread 0 of each block): 0 start,
1 neighbour flags seen (+barrier), 2 ring reloaded (+prime barrier),
3 compute done, 4 frame stores done (+barrier), 5 release issued."""
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    sys.path.insert(0, ".")
    import paper_1401_0763_b200 as P
    import sor_inputs as SI
    cfg = SI.config("C2")
    init = torch.from_numpy(cfg.init()).cuda()
    with P.Grid.create(init) as g:
        g.set_kernel("resident", int(os.environ.get("SOR_RESIDENT_T", "3")))
        g.iterate(cfg.omega, 40)
        g.iterate(cfg.omega, 180)
    sys.exit(0)
path = "/tmp/k7trace.bin"
for t in (1, 3):
    if os.path.exists(path):
        os.remove(path)
    env = dict(os.environ, SOR_RES_TRACE=path, SOR_RESIDENT_T=str(t))
    subprocess.check_call([sys.executable, __file__, "run"], env=env)
    raw = open(path, "rb").read()
    nsm = 148
    rec = 16 + 2 * nsm * 64 * 8 * 8
    blob = raw[-rec:]
    nbx, nby, npasses, T = np.frombuffer(blob[:16], dtype=np.int32)
    tr = np.frombuffer(blob[16:], dtype=np.uint64).reshape(2 * nsm, 64, 8).astype(np.int64)
    nb = nbx * nby
    P = min(npasses, 64)
    x = tr[:nb, 2:P - 1, :4]
    d = np.diff(x, axis=2)
    names = ["flags + ring in (+prime barrier)", "compute", "frame out + release"]
    print(f"T={T} blocks {nbx}x{nby}: pass {np.median(np.diff(tr[:nb, 2:P, 0], axis=1)):.0f} ns; " +
          ", ".join(f"{n} {np.median(d[:, :, i]):.0f}" for i, n in enumerate(names)))
    rel = tr[:nb, :P, 3]
    seen = tr[:nb, :P, 1]
    lat = []
    for b in range(nb):
        by, bx = divmod(b, nbx)
        for p in range(2, P - 1):
            last = max(rel[(by + dy) * nbx + bx + dx, p - 1] for dy in (-1, 0, 1) for dx in (-1, 0, 1)
                       if 0 <= by + dy < nby and 0 <= bx + dx < nbx and (dy or dx))
            lat.append(seen[b, p] - last)
    print(f"  last neighbour released -> ring in: median {np.median(lat):.0f} ns, p10 "
          f"{np.percentile(lat, 10):.0f}, p90 {np.percentile(lat, 90):.0f}")
