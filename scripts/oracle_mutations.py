"""Mutation check of the oracle's pins (test infrastructure; CPU only).

Each mutation below is a plausible mistake in oracle/oracle.c -- a dropped term, a wrong
sign or index, a transposed operand, a wrong constant.  For each, a copy of oracle/,
tests/ and the package's Python files is made under a temporary directory, the mutation
applied to the copy's oracle.c, and the oracle's CPU tests (-m "not gpu": the pins of
DESIGN.md §4, the physics checks, the round-2 readings, materials, Sod / Noh, Steinberg)
run against it.  A mutation is "killed" when at least one test fails.  The unmutated copy
must pass everything.  The GPU path is not involved.

usage: python scripts/oracle_mutations.py [out.json] [jobs]
"""
import concurrent.futures as cf
import json
import os
import re
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_physics.py", "tests/test_oracle_readings_r2.py",
         "tests/test_oracle_materials.py", "tests/test_oracle_problems.py", "tests/test_steinberg.py"]

# (name, what it breaks, old text, new text): every occurrence of old is replaced
MUTATIONS = [
    ("growth_cap_dropped", "c.5 dt <= growth * dt_prev (S:320-322)",
     "dmin(dt_cfl, p->dt_growth * c->dt_prev)", "dt_cfl"),
    ("collapse_threshold", "DT-C: dt_u < 1e-14 t",
     "dt_u < 1e-14 * tref", "dt_u < 1e-20 * tref"),
    ("viscous_speed_sign", "DT-Q: c_q = 2(c1 c + c2 (-du))",
     "2.0 * ((c1 * cs) + (c2 * (-du)))", "2.0 * ((c1 * cs) - (c2 * (-du)))"),
    ("dt_denominator", "c.5: the node speed in the signal speed",
     "(((cs + sqrt(v2)) + cq) + 1e-30)", "((cs + cq) + 1e-30)"),
    ("q_coefficients_swapped", "c.3 step 2: q = rho (c2 du^2 + c1 c |du|)",
     "rho * ((c2 * (du * du)) + ((c1 * cs) * (-du)))", "rho * ((c1 * (du * du)) + ((c2 * cs) * (-du)))"),
    ("eos_gamma", "c.3 step 1: p = (gamma - 1) rho e",
     "*p = ((gamma - 1.0) * rho) * e;", "*p = (gamma * rho) * e;"),
    ("sigma_factor", "c.3 step 3: sigma = (pf + q) / 4",
     "c->sig[K] = 0.25 * (pf + q);", "c->sig[K] = 0.5 * (pf + q);"),
    ("face_area_sign", "c.2: A = (P2 - P0) x (P3 - P1) / 2, x component",
     "f->A[0] = 0.5 * (d1[1] * d2[2] - d1[2] * d2[1]);", "f->A[0] = 0.5 * (d1[2] * d2[1] - d1[1] * d2[2]);"),
    ("face_centroid_node", "c.2: Xbar = (P0 + P1 + P2 + P3) / 4",
     "f->Xb[a] = 0.25 * (((P0[a] + P1[a]) + P2[a]) + P3[a]);",
     "f->Xb[a] = 0.25 * (((P0[a] + P1[a]) + P2[a]) + P2[a]);"),
    ("node_mass_factor", "c.3 step 5: M = sum m / 8",
     "                M = 0.125 * M;", "                M = 0.25 * M;"),
    ("ubar_weight", "c.3 step 7: ubar = (u + u') / 2",
     "ub[q] = 0.5 * (U0[h][q] + U1[h][q]);", "ub[q] = 0.5 * (U0[h][q] + U0[h][q]);"),
    ("hg_gamma_index", "HG: Gamma_1 = eta zeta",
     "case 1: return eta * zeta;", "case 1: return xi * zeta;"),
    ("hg_cap_dropped", "HG: nu = min(nu_u, (m/64)/dt)",
     "return dmin(nu_u, (m / 64.0) / dt);", "return nu_u;"),
    ("hg_work_dropped_unit", "HG: the hourglass work in the compatible energy (the per-cell entry point)",
     "(((sigma * W) + Wh) * dt)", "((sigma * W) * dt)"),
    ("hg_work_dropped_cycle", "HG: the hourglass work in the cycle's energy update",
     "((((c->sig[K] * W) + Wh) * dt) / c->m[K])", "(((c->sig[K] * W) * dt) / c->m[K])"),
    ("reflect_z", "c.3 step 6: zero normal velocity on the -z plane",
     "if (((r & 16u) && k == 0) || ((r & 32u) && k == c->nz)) v[2] = 0.0;",
     "if (((r & 32u) && k == c->nz)) v[2] = 0.0;"),
    ("donor_inverted", "c.4 step 2: the donor is the lower cell when the face moved toward +a",
     "if (!(dV > 0.0)) {", "if (dV > 0.0) {"),
    ("donor_velocity_mean", "c.4 step 2: Ubar_D = sum of the 8 nodes' u' / 8",
     "Ub[q] = 0.125 * s;", "Ub[q] = 0.25 * s;"),
    ("momentum_remap_term", "c.4 step 4: u'' = u' + (D_P - u' D_m) / M''",
     "un[q] = u1 + ((DP[q] - (u1 * Dm)) / M2);", "un[q] = u1 + (DP[q] / M2);"),
    ("sedov_deposit", "c.6: e_000 = E0 / m_000",
     "c->e[0] = p->e_deposit / c->m[0];", "c->e[0] = p->e_deposit;"),
    ("steinberg_eta_exponent", "Fig. 6b: eta^(1/3)",
     "pow(eta, 1.0 / 3.0)", "pow(eta, 1.0 / 2.0)"),
    # multi-material cells (DESIGN.md §10d readings MM1-MM6)
    ("mm_material_density", "MM1: rho_m = m_m / (f_m V)",
     "double rk = mm[k] / (f[k] * V);", "double rk = mm[k] / V;"),
    ("mm_sound_speed_gamma", "MM1: c = sqrt(sum f_m gamma_m pf_m / rho)",
     "g = f[k] * (gam[k] * pfk);", "g = f[k] * pfk;"),
    ("mm_volume_flux", "MM5: phi_m = f_m,D dV",
     "o->phim[m] = c->mf[m][D] * dV;", "o->phim[m] = (c->mmat[m][D] / c->V1[D]) * dV;"),
    ("mm_energy_remap", "MM6: e''_m = e'_m + (dE_m - e'_m dm_m) / m''_m",
     "e1 + ((c->dEm[m][K] - (e1 * c->dmm[m][K])) / mm2)", "e1 + (c->dEm[m][K] / mm2)"),
    ("mm_fraction_normalisation", "MM6: f''_m = V''_m / sum_k V''_k",
     "c->mf[m][K] = c->vm2[m][K] / VV;", "c->mf[m][K] = c->vm2[m][K] / c->V1[K];"),
    ("mm_energy_share", "MM4: each material does the work on its share f_m",
     "c->e1m[m][K] = em - (((((sm * W) + Wh) * dt) * f) / mm);", "c->e1m[m][K] = em - ((((sm * W) + Wh) * dt) / mm);"),
]


def copy_tree(dst):
    for d in ("oracle", "tests", "paper_2209_01983_b200"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(dst, d),
                        ignore=shutil.ignore_patterns("*.so", "*.o", "lib", "__pycache__", "golden_big*"))


def run(name, old, new):
    d = tempfile.mkdtemp(prefix=f"mut_{name}_")
    try:
        copy_tree(d)
        src = os.path.join(d, "oracle", "oracle.c")
        text = open(src).read()
        n = text.count(old) if old else 0
        if old:
            if n == 0:
                return {"mutation": name, "error": "pattern not found"}
            open(src, "w").write(text.replace(old, new))
        t0 = time.time()
        # (a test running past 300 s -- a mutated scheme gone unstable -- ends the run: killed)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                            "--timeout", "300", "--timeout-method", "thread", *TESTS],
                           cwd=d, capture_output=True, text=True, timeout=3600)
        tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        failed = int(m.group(1)) if (m := re.search(r"(\d+) failed", tail)) else 0
        errors = int(m.group(1)) if (m := re.search(r"(\d+) error", tail)) else 0
        passed = int(m.group(1)) if (m := re.search(r"(\d+) passed", tail)) else 0
        killing = sorted({ln.split("::")[1].split(" ")[0].split("[")[0]
                          for ln in r.stdout.splitlines() if ln.startswith("FAILED ") and "::" in ln})
        if r.returncode and not killing:  # timed out (the thread method ends the run) or crashed
            killing = ["(a test ran past the 300-s limit: the mutated scheme does not finish)"
                       if "Timeout" in r.stdout + r.stderr else "(the run crashed)"]
        return {"mutation": name, "sites": n, "failed": failed, "errors": errors, "passed": passed,
                "killed": r.returncode != 0, "returncode": r.returncode, "killing_tests": killing,
                "seconds": round(time.time() - t0, 1), "summary": tail[-300:]}
    finally:
        shutil.rmtree(d, ignore_errors=True)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    jobs = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count() or 4
    cases = [("none", "the unmutated oracle", "", "")] + MUTATIONS
    res = {}
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        futs = {ex.submit(run, name, old, new): (name, what) for name, what, old, new in cases}
        for f in cf.as_completed(futs):
            name, what = futs[f]
            r = f.result()
            r["breaks"] = what
            res[name] = r
            print(json.dumps(r), flush=True)
    base = res.pop("none")
    killed = sum(1 for r in res.values() if r.get("killed"))
    summary = {"baseline": base, "mutations": [res[n] for n, *_ in MUTATIONS], "killed": killed,
               "total": len(MUTATIONS), "tests": TESTS}
    print(json.dumps({"killed": killed, "total": len(MUTATIONS), "baseline_passed": base.get("passed"),
                      "baseline_failed": base.get("failed")}))
    if out:
        with open(out, "w") as fh:
            json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
