"""Mutation check of the oracle's pins: each mutation is a plausible mistake in
oracle/oracle.c (a reversed order, a dropped term, a wrong sign, a transposed operand).  For each one
a scratch copy of oracle/ + synth/ + tests/ is made under /tmp, the mutation applied, and the
CPU pins (tests/test_oracle_pins.py) run; a mutation that leaves every pin green is a hole.

usage: python scripts/oracle_mutations.py [--out profiles/r02_oracle_mutations.md]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, exact source text, replacement) — each applied alone
MUTATIONS = [
    ("depth order reversed (cmp_cand)",
     "if (x->key != y->key) return x->key < y->key ? -1 : 1;",
     "if (x->key != y->key) return x->key > y->key ? -1 : 1;"),
    ("orderable key without the sign flip",
     "return (u & 0x80000000u) ? ~u : (u | 0x80000000u);",
     "return u ^ 0x80000000u;"),
    ("Hessian: -Q term dropped (sigma Q d d^T Q only)",
     "H[3 * a + b] = sigma * (U[a] * U[b] - PQP);",
     "H[3 * a + b] = sigma * (U[a] * U[b]);"),
    ("Hessian: sign of the -Q term flipped",
     "H[3 * a + b] = sigma * (U[a] * U[b] - PQP);",
     "H[3 * a + b] = sigma * (U[a] * U[b] + PQP);"),
    ("Hessian: P transposed in U (P_{a,0} -> P_{0,a} index)",
     "U[a] = g->P[a] * u0 + g->P[3 + a] * u1;",
     "U[a] = g->P[a] * u1 + g->P[3 + a] * u0;"),
    ("compositing: T updated with sigma instead of the clamped alpha",
     "const double Tn = T * (1.0 - alpha);",
     "const double Tn = T * (1.0 - sigma);"),
    ("backward: colour-behind B updated before dL/dalpha is formed",
     "const double ga = rc->T * gsum;",
     "for (int ch = 0; ch < 3; ++ch) Bc[ch] = rc->alpha * g->col[ch] + (1 - rc->alpha) * Bc[ch];\n          gsum = 0; for (int ch = 0; ch < 3; ++ch) gsum += dLdC[ch] * (g->col[ch] - Bc[ch]);\n          const double ga = rc->T * gsum;"),
    ("backward: S weighted by dL/dalpha without sigma",
     "contrib[14] = ga * H[0];",
     "contrib[14] = ga * H[0] / (sg > 0 ? sg : 1);"),
    ("backward: opacity gradient without the sigmoid derivative",
     "contrib[10] = ga * sg * (1.0 - g->o);",
     "contrib[10] = ga * sg;"),
    ("termination compares T before the update (T < t_min)",
     "if (Tn < tmin) break;",
     "if (T < tmin) break;"),
]


def run(mutations, timeout=900):
    rows = []
    for name, a, b in mutations:
        d = tempfile.mkdtemp(prefix="orcmut_")
        try:
            for sub in ("oracle", "synth", "tests"):
                shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                                ignore=shutil.ignore_patterns("*.so", "__pycache__", "_build"))
            path = os.path.join(d, "oracle", "oracle.c")
            src = open(path).read()
            if src.count(a) < 1:
                rows.append((name, "not applicable (text not found)", ""))
                continue
            open(path, "w").write(src.replace(a, b, 1))
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-p", "no:cacheprovider"],
                               cwd=d, capture_output=True, text=True, timeout=timeout)
            failed = [ln.split("::", 1)[1].split(" ")[0] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
            rows.append((name, "caught" if failed else "NOT CAUGHT", f"{tail}; first failing: {failed[:3]}"))
        finally:
            shutil.rmtree(d, ignore_errors=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = run(MUTATIONS)
    lines = ["| mutation of oracle/oracle.c | result | pins |", "|---|---|---|"]
    lines += [f"| {n} | {r} | {t} |" for n, r, t in rows]
    txt = "\n".join(lines)
    print(txt)
    if args.out:
        with open(args.out, "w") as f:
            f.write("# Oracle mutation check (scripts/oracle_mutations.py)\n\n" + txt + "\n")
    return 0 if all(r != "NOT CAUGHT" for _, r, _ in rows) else 1


if __name__ == "__main__":
    sys.exit(main())
