"""Mutation check of the oracle pins.

Copies oracle/, sor_inputs/ and the CPU pin tests into a scratch directory,
applies one mutation at a time to oracle/sor_oracle.c, rebuilds it there and
runs the pins.  Every mutation must make at least one pin fail.  Usage:
    python tools/mutate_oracle.py [--out profiles/r2_oracle_mutations.txt]
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, [(old, new), ...]) applied to sor_oracle.c; `old` must occur.
MUTATIONS = [
    ("phase: fp32 update in double, rounded once",
     [("        T s = (up[j] + dn[j]) + (uc[j - 1] + uc[j + 1]);                      \\\n"
       "        T a = q * s;                                                          \\\n"
       "        T r = a - uc[j];                                                      \\\n"
       "        T un = uc[j] + w * r;                                                 \\\n",
       "        double s = ((double)up[j] + dn[j]) + ((double)uc[j - 1] + uc[j + 1]); \\\n"
       "        double a = (double)q * s;                                             \\\n"
       "        double r = a - uc[j];                                                 \\\n"
       "        T un = (T)(uc[j] + (double)w * r);                                    \\\n")]),
    ("jacobi: fp32 in double + sum order (N+W)+S+E",
     [("          T s = (c[-ld] + c[ld]) + (c[-1] + c[1]);     /* (N+S)+(W+E) */          \\\n"
       "          T a = q * s;                                                            \\\n",
       "          double s = (((double)c[-ld] + c[-1]) + c[ld]) + c[1];                   \\\n"
       "          T a = (T)((double)q * s);                                               \\\n")]),
    ("jacobi: fp32 in double, rounded once (sum order kept)",
     [("          T s = (c[-ld] + c[ld]) + (c[-1] + c[1]);     /* (N+S)+(W+E) */          \\\n"
       "          T a = q * s;                                                            \\\n",
       "          double s = ((double)c[-ld] + c[ld]) + ((double)c[-1] + c[1]);           \\\n"
       "          T a = (T)((double)q * s);                                               \\\n")]),
    ("sor3d: fp32 in double, rounded once",
     [("          T s = ((uc[-lx] + uc[lx]) + (uc[-1] + uc[1])) + (uc[-lp] + uc[lp]);   \\\n"
       "          T a = s / six;                                                         \\\n"
       "          T r = a - uc[0];                                                       \\\n"
       "          T un = uc[0] + w * r;                                                  \\\n",
       "          double s = (((double)uc[-lx] + uc[lx]) + ((double)uc[-1] + uc[1])) + ((double)uc[-lp] + uc[lp]); \\\n"
       "          double a = s / 6.0;                                                    \\\n"
       "          double r = a - uc[0];                                                  \\\n"
       "          T un = (T)(uc[0] + (double)w * r);                                     \\\n")]),
    ("sor3d: a = s * (1/6) instead of s / 6 (reading N3-1)",
     [("          T a = s / six;                                                         \\\n",
       "          T a = s * ((T)1 / six);                                                \\\n")]),
    ("phase: colours swapped",
     [("const int64_t j0 = (((row_off + i + 1) & 1) == c) ? 1 : 2;",
       "const int64_t j0 = (((row_off + i) & 1) == c) ? 1 : 2;")]),
    ("phase: sum order (N+W)+(S+E)",
     [("T s = (up[j] + dn[j]) + (uc[j - 1] + uc[j + 1]);",
       "T s = (up[j] + uc[j - 1]) + (dn[j] + uc[j + 1]);")]),
    ("phase: |delta| as |w*r|",
     [("T d = ABS(un - uc[j]);", "T d = ABS(w * r);")]),
    ("run: <= instead of < in the stop test",
     [("if (mode == 1 && (double)m < tol) {                /* P:327 */",
       "if (mode == 1 && (double)m <= tol) {               /* P:327 */")]),
]

TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_rounding_pins.py"]


def run(mut_name, edits, base):
    work = tempfile.mkdtemp(prefix="orcmut_")
    try:
        for d in ("oracle", "sor_inputs", "tests"):
            shutil.copytree(os.path.join(base, d), os.path.join(work, d),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        shutil.copy(os.path.join(base, "pytest.ini"), work)
        src = os.path.join(work, "oracle", "sor_oracle.c")
        text = open(src).read()
        for old, new in edits:
            if old not in text:
                return f"{mut_name}: PATTERN NOT FOUND"
            text = text.replace(old, new)
        open(src, "w").write(text)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *TESTS],
                           cwd=work, capture_output=True, text=True, timeout=1800)
        tail = [ln for ln in r.stdout.splitlines() if " passed" in ln or " failed" in ln]
        return f"{mut_name}: {tail[-1] if tail else r.stdout[-300:]}"
    finally:
        shutil.rmtree(work, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    lines = [run("(none: unmutated oracle)", [], ROOT)]
    for name, edits in MUTATIONS:
        lines.append(run(name, edits, ROOT))
        print(lines[-1], flush=True)
    txt = "\n".join(lines) + "\n"
    print(txt)
    if a.out:
        open(a.out, "w").write(txt)


if __name__ == "__main__":
    main()
