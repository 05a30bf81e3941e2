"""Time crk_pm_accel on c4 (2x256^3 particles, 256^3 mesh) with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import make_config
from paper_2310_16122_b200 import PM

parts, params = make_config("c4")
dev = torch.device("cuda", 0)
t = lambda k: torch.from_numpy(np.ascontiguousarray(parts[k])).to(dev)  # noqa: E731
x, y, z, m = t("x"), t("y"), t("z"), t("m")
rs = float(np.sqrt(params["rcut2"])) / 4.5
for ng in (256, 512):
    pm = PM(ng, params["box"], rs, 1.0)
    for _ in range(2):
        pm.accel(x, y, z, m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pm.accel(x, y, z, m)
    e1.record()
    torch.cuda.synchronize()
    print(f"PM {ng}^3 mesh, {x.shape[0]} particles: {e0.elapsed_time(e1) / 5:.2f} ms")
    pm.close()

# slab-decomposed sequence on one GPU (P = 1: the collectives are no-op copies), per phase
from paper_2310_16122_b200 import SlabPM  # noqa: E402
from paper_2310_16122_b200.pm_dist import pm_accel_emulated  # noqa: E402

for ng in (256, 512):
    spm = SlabPM(ng, params["box"], rs, 1.0, 0, 1)
    for _ in range(2):
        pm_accel_emulated([spm], [(x, y, z, m)])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pm_accel_emulated([spm], [(x, y, z, m)])
    e1.record()
    torch.cuda.synchronize()
    print(f"slab PM (P=1) {ng}^3 mesh: {e0.elapsed_time(e1) / 5:.2f} ms (includes the emulated collectives' copies)")
    spm.close()
