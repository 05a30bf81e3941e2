"""Mutation check of the oracle's pins (VERDICT r1 "what's missing" 1).

Each mutation is a plausible misreading or typo of one step of oracle/oracle.c (a wrong
sign, a dropped term, a swapped operand, a different softening or limiter form).  For
each one a mutated copy of oracle.c is compiled to a temporary library and the oracle
pins (tests/test_oracle_pins.py) are run against it through CRK_ORACLE_LIB; the mutation
is KILLED when at least one pin fails.  A surviving mutation means the pins cannot tell
that reading from the one the oracle implements.

    python tools/mutation_check.py [--jobs 4] [--only name,...]

Exit code 0 when every mutation is killed, 1 otherwise.  tests/test_mutations.py runs it.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")
PINS = [os.path.join(ROOT, "tests", "test_oracle_pins.py"), os.path.join(ROOT, "tests", "test_subcycle.py")]

# (name, what it misreads, original text, replacement); the original must occur exactly once
MUTATIONS = [
    ("av_mu_clamp", "AV mu = max(0, .) instead of min(0, .) (O9)",
     "if (mu > 0.0) mu = 0.0;", "if (mu < 0.0) mu = 0.0;"),
    ("av_linear_sign", "AV linear term +C_l c mu instead of -C_l c mu (O9)",
     "Q += rk[s] * (-Cl * ck[s] * mu + Cq * mu * mu);", "Q += rk[s] * (Cl * ck[s] * mu + Cq * mu * mu);"),
    ("vanleer_phi_one", "limiter forced to phi = 1 (O9)",
     "phi = 4.0 * rr / ((1.0 + rr) * (1.0 + rr));", "phi = 1.0;"),
    ("vanleer_classic_form", "limiter 2r/(1+r) instead of 4r/(1+r)^2 (O9)",
     "phi = 4.0 * rr / ((1.0 + rr) * (1.0 + rr));", "phi = 2.0 * rr / (1.0 + rr);"),
    ("sound_speed", "c = sqrt(gamma P rho) instead of sqrt(gamma P / rho) (O8)",
     "cs[t] = sqrt(gam * P[t] / r_);", "cs[t] = sqrt(gam * P[t] * r_);"),
    ("plummer_on_r", "softening (r + eps)^-3 instead of (r^2 + eps^2)^-3/2 (O5)",
     "double newton = pow(s + (double)p->eps2, -1.5);",
     "double newton = pow(sqrt(s) + sqrt((double)p->eps2), -3.0);"),
    ("poly_sign", "grid polynomial added instead of subtracted (O5)",
     "double f = newton - poly;", "double f = newton + poly;"),
    ("energy_split", "du/dt with (P_i + Q) instead of (P_i + Q/2) (O9)",
     "(P[i] + 0.5 * Q)", "(P[i] + Q)"),
    ("av_eta_own_h", "AV eta_k with H_i for both particles instead of H_k (O9)",
     "const double Hk[2] = {H[i], H[j]};", "const double Hk[2] = {H[i], H[i]};"),
    ("gij_sign", "G_ij = (grad W_ij + grad W_ji)/2 instead of the difference (O9)",
     "G[k] = 0.5 * (gij[k] - gji[k]);", "G[k] = 0.5 * (gij[k] + gji[k]);"),
    ("accel_mass", "m_j instead of m_i on the left of the momentum equation (O9)",
     "double fa = -VV * (P[i] + P[j] + Q) / (double)m[i];", "double fa = -VV * (P[i] + P[j] + Q) / (double)m[j];"),
    ("density_mass", "rho_i = sum m_i W^R_ij instead of m_j (O8)",
     "r_ += (double)m[j] * WR;", "r_ += (double)m[i] * WR;"),
    ("eos_gamma", "P = gamma rho u instead of (gamma - 1) rho u (O8)",
     "P[t] = (gam - 1.0) * r_ * (double)u[i];", "P[t] = gam * r_ * (double)u[i];"),
    ("grad_w_sign", "kernel gradient with the wrong sign (O6)",
     "return -(56.0 / 3.0) * sigma / pow(H, 5)", "return (56.0 / 3.0) * sigma / pow(H, 5)"),
    ("no_self_term", "self term left out of the gather sums (O2/O6)",
     "if (j == i) return pred == PRED_GATHER_SELF;", "if (j == i) return 0;"),
    ("dm1_delta", "delta_ag m0 term of grad m1 dropped (O7)",
     "dm1[a][a] += m0;", "dm1[a][a] += 0.0 * m0;"),
    ("dB_drops_dm2", "(grad m2) B term of grad B dropped (O7)",
     "rhs[a] += dm2[a][b][g] * Bi[b];", "rhs[a] += 0.0 * dm2[a][b][g] * Bi[b];"),
    ("corrected_grad_B_term", "B^g W term of grad W^R dropped (O7)",
     "A * (dBd + B[gg]) * W", "A * dBd * W"),
    ("kick_sign", "gravity kick v - dt a (O5)",
     "vout[3 * t + 0] = (double)vx[i] + dt * a[0];", "vout[3 * t + 0] = (double)vx[i] - dt * a[0];"),
    ("predicate_le", "gravity predicate s32 <= rcut2 instead of strict (O2)",
     "case PRED_GRAV: return s < c->rcut2;", "case PRED_GRAV: return s <= c->rcut2;"),
    ("list_no_slack", "leaf-pair test without the 2^-20 slack (O4)",
     "return d2 < cut2 * (1.0 + ldexp(1.0, -20));", "return d2 < cut2;"),
    ("predicate_fp64", "membership decided on the fp64 s instead of the fp32 fma sequence (O2)",
     "float t = fx * fx;", "double t = (double)fx * fx + (double)fy * fy + (double)fz * fz; return (float)t;"),
    ("wendland_sigma_c2", "W normalised with Wendland C2's 21/(2 pi) instead of C4's 495/(32 pi) (O6)",
     "return sigma / (H * H * H) * pow(t, 6)", "return 21.0 / (2.0 * ORC_PI) / (H * H * H) * pow(t, 6)"),
    ("wendland_c2_shape", "W of Wendland C2 shape (1-q)^4 (1 + 4q) instead of C4 (O6)",
     "pow(t, 6) * (1.0 + 6.0 * q + 35.0 * q * q / 3.0)", "pow(t, 4) * (1.0 + 4.0 * q)"),
    ("no_min_image", "periodic differences without the minimum image (O1)",
     "if (d > 0.5 * L) d -= L;", "if (0) d -= L;"),
    ("drift_truncate", "drift rounded toward zero instead of to the nearest lattice point (sub-cycle)",
     "float r = rintf(t / q) * q;", "float r = truncf(t / q) * q;"),
    ("courant_no_cfl", "Courant limit H / c without the C_cfl factor (sub-cycle)",
     "const double dc = c_cfl * (double)H[i] / (double)cs[i];", "const double dc = (double)H[i] / (double)cs[i];"),
    ("knn_off_by_one", "H from the (k+1)-th instead of the k-th neighbour distance (sub-cycle)",
     "const float d2 = m >= k ? d[k - 1] : INFINITY;", "const float d2 = m > k ? d[k] : INFINITY;"),
]


def _gcc_flags():
    sys.path.insert(0, ROOT)
    import oracle

    return list(oracle.CFLAGS)


def run_one(m, tmp, flags, timeout=600):
    name, why, old, new = m
    src = open(SRC).read()
    if src.count(old) != 1:
        return name, "error", f"original text occurs {src.count(old)} times"
    mdir = os.path.join(tmp, name)
    os.makedirs(mdir, exist_ok=True)
    c = os.path.join(mdir, "oracle.c")
    so = os.path.join(mdir, "liboracle.so")
    open(c, "w").write(src.replace(old, new))
    r = subprocess.run(["gcc", *flags, "-o", so, c, "-lm"], capture_output=True, text=True)
    if r.returncode != 0:
        return name, "error", "compile: " + r.stderr[-300:]
    env = dict(os.environ, CRK_ORACLE_LIB=so, OMP_NUM_THREADS="2")
    t0 = time.time()
    r = subprocess.run([sys.executable, "-m", "pytest", *PINS, "-m", "not gpu", "-x", "-q", "-p", "no:cacheprovider"],
                       capture_output=True, text=True, cwd=ROOT, env=env, timeout=timeout)
    failed = [ln.split("::", 1)[1].split(" ")[0] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
    status = "killed" if r.returncode == 1 and failed else ("survived" if r.returncode == 0 else "error")
    detail = failed[0] if failed else r.stdout[-300:]
    return name, status, f"{detail} ({time.time() - t0:.0f} s)"


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=max(1, min(6, (os.cpu_count() or 2) // 2)))
    ap.add_argument("--only", default="")
    ap.add_argument("--json", default="")
    a = ap.parse_args(argv)
    muts = [m for m in MUTATIONS if not a.only or m[0] in a.only.split(",")]
    flags = _gcc_flags()
    res = []
    with tempfile.TemporaryDirectory() as tmp, cf.ThreadPoolExecutor(a.jobs) as ex:
        for name, status, detail in ex.map(lambda m: run_one(m, tmp, flags), muts):
            why = next(m[1] for m in MUTATIONS if m[0] == name)
            print(f"{status:8s} {name:22s} {why}  <- {detail}", flush=True)
            res.append(dict(name=name, what=why, status=status, detail=detail))
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)
    bad = [r for r in res if r["status"] != "killed"]
    print(f"{len(res) - len(bad)}/{len(res)} mutations killed")
    return 0 if not bad else 1


if __name__ == "__main__":
    sys.exit(main())
