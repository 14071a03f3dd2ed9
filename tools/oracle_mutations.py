#!/usr/bin/env python
"""Plant mutations in a copy of oracle/oracle.cpp and check that the CPU pins
catch each one (VERDICT r01 "Next round" #1).  Writes
profiles/r02/oracle_mutations.txt.  Test infrastructure only."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()

MUTATIONS = [
    ("camera centre C = -R t (not -R^T t)",
     "v += (double)c.R[r * 3 + a] * (double)c.t[r];", "v += (double)c.R[a * 3 + r] * (double)c.t[r];"),
    ("view direction reversed (C - mu)",
     "dir[q] = (double)mu[q] - (double)rk.C[q];", "dir[q] = (double)rk.C[q] - (double)mu[q];"),
    ("colour clamp removed",
     "c->col[3 * r + q] = (float)std::max(rgb[q], 0.0);", "c->col[3 * r + q] = (float)rgb[q];"),
    ("conic B sign flipped",
     "c->conB[r] = -b / det;", "c->conB[r] = b / det;"),
    ("conic A <-> C swapped",
     "c->conA[r] = cc / det; c->conB[r] = -b / det; c->conC[r] = a / det;",
     "c->conA[r] = a / det; c->conB[r] = -b / det; c->conC[r] = cc / det;"),
    ("cluster id shifted in the key",
     "((uint64_t)k << 32) | (uint64_t)dbits;", "((uint64_t)k << 33) | (uint64_t)dbits;"),
    ("degenerate cull removed",
     "    return det > 0.0f;\n}", "    return true;\n}"),
    ("O7 right extreme uses -dyR",
     "float right = mx + ((dlo <= dyR && dyR <= dhi) ? ex : mxf(xr(dlo), xr(dhi)));",
     "float right = mx + ((dlo <= dyL && dyL <= dhi) ? ex : mxf(xr(dlo), xr(dhi)));"),
]
TESTS = ["tests/test_oracle_wholepath.py", "tests/test_oracle_shading.py",
         "tests/test_oracle_geometry.py", "tests/test_oracle_pipeline.py"]


def main():
    out = ["# planted oracle mutations vs the CPU pins (-m 'not gpu' oracle tests)",
           "# mutation | caught | first failing tests", ""]
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    ok_all = True
    for name, old, new in MUTATIONS:
        assert SRC.count(old) == 1, name
        path = os.path.join(tmp, f"m{len(out)}.cpp")
        open(path, "w").write(SRC.replace(old, new))
        env = dict(os.environ, CR_ORACLE_MUTANT_SRC=path)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                            *TESTS], cwd=ROOT, env=env, capture_output=True, text=True)
        failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
        if r.returncode < 0:  # the mutant crashed the test process (e.g. out-of-range slot)
            failed.append(f"crash::signal {-r.returncode} after {r.stdout.count('F')} failures")
        caught = r.returncode != 0 and bool(failed)
        ok_all &= caught
        out.append(f"{name} | {'CAUGHT' if caught else 'MISSED'} | "
                   + ", ".join(f.split("::")[-1] for f in failed[:4]))
        print(out[-1], flush=True)
    dst = os.path.join(ROOT, "profiles", "r02", "oracle_mutations.txt")
    open(dst, "w").write("\n".join(out) + "\n")
    return 0 if ok_all else 1


if __name__ == "__main__":
    sys.exit(main())
