"""Print GPU-vs-oracle error statistics per field (diagnostic; uses the oracle)."""
import sys, os, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle
from crk_testutil import cached_config, run_gpu

def report(name):
    parts, params = cached_config(name)
    g = run_gpu(parts, params)
    ref = oracle.substep(parts, params)
    gi = g["in"]; T = ref["targets"]
    out = {"config": name}
    def st(e):
        e = np.asarray(e, np.float64).ravel()
        return dict(max=float(e.max()), p99=float(np.quantile(e, 0.99)), med=float(np.median(e)))
    a = np.stack([gi["ax"], gi["ay"], gi["az"]], 1)
    out["grav"] = st(np.linalg.norm(a - ref["grav_a"], axis=1) / ref["grav_S"])
    for k in ("V", "A", "rho", "P", "cs"):
        out[k] = st(np.abs(gi[k][T] - ref[k]) / np.abs(ref[k]))
    for k in ("B", "dA", "dB", "dv"):
        r = ref[k]; gg = gi[k][:, T].T
        out[k] = st(np.abs(gg - r) / max(np.abs(r).max(), 1e-300))
    ah = np.stack([gi["ahx"], gi["ahy"], gi["ahz"]], 1)[T]
    out["ah"] = st(np.linalg.norm(ah - ref["a"], axis=1) / ref["Sa"])
    S = ref["Sdu"]; ok = S > 0
    out["du"] = st(np.abs(gi["dudt"][T][ok] - ref["dudt"][ok]) / S[ok]) if ok.any() else None
    print(json.dumps(out))

for n in sys.argv[1:]:
    report(n)
