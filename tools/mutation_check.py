#!/usr/bin/env python
"""Mutation check of the oracle's pins (VERDICT r1 "What's weak" #1): apply one plausible
mistake at a time to oracle/hj_oracle.c, rebuild, run the CPU pins, and report whether
at least one pin fails.  The source is restored afterwards (try/finally).

    python tools/mutation_check.py > profiles/r2/oracle_mutations.txt
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "hj_oracle.c")
LIB = os.path.join(ROOT, "oracle", "_hj_oracle.so")

MUTATIONS_ALL = [
    ("speed ignored", "    if (!p->speed) return 1.0;\n", "    return 1.0;\n"),
    ("speed squared", "    return or_interp_field(p, p->speed, gi, 1.0);",
     "    double c_ = or_interp_field(p, p->speed, gi, 1.0); return c_ * c_;"),
    ("margin sign flipped", "    if (margin) *margin = second - best;",
     "    if (margin) *margin = best - second;"),
    ("margin zero", "    if (margin) *margin = second - best;", "    if (margin) *margin = 0.0;"),
    ("geo never updated (rounding)", "            if (dist < mg) mg = dist;", ""),
    ("geo never updated (box gap)", "                if (gap < mg) mg = gap;", ""),
    ("highest-index argmin", "        if (v < best) {", "        if (v <= best) {"),
    ("R10: other pieces' targets outside S_k stay targets",
     "        if (!in) cls[i] = OR_GHOST;",
     "        if (!in) cls[i] = (p->piece[i] >= 0) ? OR_TARGET : OR_GHOST;"),
    ("R8: feedback at the nearest node", "        or_min_bracket(p, V, gi, &a, &margin);",
     "        double gr_[3] = {(double)r[0], (double)r[1], (double)r[2]};\n"
     "        or_min_bracket(p, V, gr_, &a, &margin);"),
    ("RA < instead of <=", "fabs(Vi[i][j] - V[j]) <= thr", "fabs(Vi[i][j] - V[j]) < thr"),
    ("step budget +1", "        if (s >= n_max) break;", "        if (s > n_max) break;"),
    ("step budget -1", "        if (s >= n_max) break;", "        if (s + 1 >= n_max) break;"),
    ("label rounding floor(g)", "            double t = gi[d] + 0.5;", "            double t = gi[d];"),
    ("assembly max", "                if (!any || Vk[k][j] < v) v = Vk[k][j];",
     "                if (!any || Vk[k][j] > v) v = Vk[k][j];"),
    ("prolongation radius -1", "            long reach = ratio[d] + band;",
     "            long reach = ratio[d] + band - 1;"),
    ("label -1 -> no bits", "        else cm[j] = pieces;", "        else cm[j] = 0ull;"),
    ("label -1 -> the exit set too", "        else cm[j] = pieces;",
     "        else cm[j] = pieces | (exit_set ? (1ull << m) : 0ull);"),
    ("label -2 -> all sets", "        else if (l == -2) cm[j] = exit_set ? (1ull << m) : 0ull;",
     "        else if (l == -2) cm[j] = pieces | (1ull << m);"),
    ("exit test strict", "if (labels[j] == -1 && Vc[j] >= Vexit[j] - tol) labels[j] = -2;",
     "if (labels[j] == -1 && Vc[j] > Vexit[j] - tol) labels[j] = -2;"),
    ("exit test on labelled nodes", "if (labels[j] == -1 && Vc[j] >= Vexit[j] - tol) labels[j] = -2;",
     "if (labels[j] < 0 || Vc[j] >= Vexit[j] - tol) labels[j] = -2;"),
    ("box tolerance 1e-2", "#define OR_BOX_EPS 1e-6", "#define OR_BOX_EPS 1e-2"),
    ("beta = exp(-lambda h)", "return 1.0 / (1.0 + p->lam * p->h);", "return exp(-p->lam * p->h);"),
    ("Kruzkov cost dropped", "(p->cost == OR_COST_KRUZKOV) ? (1.0 - beta)",
     "(p->cost == OR_COST_KRUZKOV) ? 0.0"),
    ("foot x - h f", "foot[d] = gi[d] + p->h * f[d] / or_spacing(p, d);",
     "foot[d] = gi[d] - p->h * f[d] / or_spacing(p, d);"),
    ("interp weights swapped", "                wt *= w[d];\n", "                wt *= 1.0 - w[d];\n"),
    ("drift A transposed", "s += p->A[3 * d + e] * x[e];", "s += p->A[3 * e + d] * x[e];"),
    ("running cost |a|^2 dropped", "+ p->lr * a2;", ";"),
    ("stopping rule <=", "        if (res < tol) break;", "        if (res <= tol * 10) break;"),
    ("target piece label of wrong node", "        int pc = p->piece[or_flatten(p, r)];",
     "        int pc = p->piece[or_flatten(p, r) > 0 ? or_flatten(p, r) - 1 : 0];"),
    ("Dubins heading sign", "f[2] = p->dub_w * a[0];", "f[2] = -p->dub_w * a[0];"),
]

MUTATIONS = [m for m in MUTATIONS_ALL if not os.environ.get("ONLY") or os.environ["ONLY"] in m[0]]

TESTS = ["tests/test_oracle_pins.py", "tests/test_parallel_gloo.py"]


def main():
    orig = open(SRC).read()
    results = []
    try:
        for name, old, new in MUTATIONS:
            if orig.count(old) < 1:
                results.append((name, "PATTERN NOT FOUND"))
                continue
            open(SRC, "w").write(orig.replace(old, new))
            if os.path.exists(LIB):
                os.remove(LIB)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                                *TESTS], cwd=ROOT, capture_output=True, text=True, timeout=1800)
            failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED")]
            if not r.returncode:
                verdict = "NOT CAUGHT"
            elif failed:
                verdict = "caught by " + failed[0].split("::")[-1].split(" ")[0]
            else:
                verdict = "ERROR (did not build/collect): " + r.stdout[-200:].replace("\n", " ")
            results.append((name, verdict))
            print(f"{name:55s} {verdict}", flush=True)
    finally:
        open(SRC, "w").write(orig)
        if os.path.exists(LIB):
            os.remove(LIB)
        subprocess.run([sys.executable, "-c", "import oracle; oracle.build()"], cwd=ROOT, check=True)
    missed = [n for n, v in results if not v.startswith("caught")]
    print(f"\n{len(results) - len(missed)} of {len(results)} mutations caught; missed: {missed}")
    return 1 if missed else 0


if __name__ == "__main__":
    sys.exit(main())
