"""Mutation check of the oracle's GA pins (VERDICT r1 "Next" item 1).

Applies one plausible slip at a time to a copy of oracle/ffs_oracle.c, builds
it under /tmp, and runs the hand-derived GA goldens (tests/test_oracle_ga_ops.py)
plus the paper-operator pins against it.  Every perturbation must turn the
suite red; the unmodified source must pass.  CPU only:

    python scripts/perturb_oracle.py
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "ffs_oracle.c")

PERTURBATIONS = {
    "selection: N and S swapped": (
        "                   ((row + h - 1) % h) * w + col,      /* N: row above */\n"
        "                   ((row + 1) % h) * w + col,          /* S: row below */",
        "                   ((row + 1) % h) * w + col,          /* S: row below */\n"
        "                   ((row + h - 1) % h) * w + col,      /* N: row above */"),
    "selection: E and W swapped": (
        "                   row * w + (col + 1) % w,            /* E: next column */\n"
        "                   row * w + (col + w - 1) % w};       /* W: previous column */",
        "                   row * w + (col + w - 1) % w,        /* W: previous column */\n"
        "                   row * w + (col + 1) % w};           /* E: next column */"),
    "selection: ties to the last candidate": (
        "if (fit[nb[t]] > fit[best]) best = nb[t];", "if (fit[nb[t]] >= fit[best]) best = nb[t];"),
    "selection: no torus (clamped edges)": (
        "((row + h - 1) % h) * w + col,      /* N: row above */",
        "(row > 0 ? row - 1 : row) * w + col, /* N: row above */"),
    "argmax: ties to the last cell": (
        "if (fit[i] > fit[b]) b = i;", "if (fit[i] >= fit[b]) b = i;"),
    "argmin: ties to the last cell": (
        "if (fit[i] < fit[w]) w = i;", "if (fit[i] <= fit[w]) w = i;"),
    "replacement: history on >= instead of >": (
        "if (fit[b] > hfit[li]) {", "if (fit[b] >= hfit[li]) {"),
    "replacement: worst taken before the history update sees the best": (
        "    size_t wst = base + or_argmin_fitness(fit + base, tile);\n    memcpy(X + wst * cells, HX",
        "    size_t wst = base + or_argmax_fitness(fit + base, tile);\n    memcpy(X + wst * cells, HX"),
    "migration: ring runs I <- I+1": (
        "const char *src = li == 0 ? incoming : donors + rec * (li - 1);",
        "const char *src = donors + rec * ((li + 1) % nisl);"),
    "migration: shard imports from rank+1": (
        "all + rec * ((rank + world - 1) % world)", "all + rec * ((rank + 1) % world)"),
    "migration: sequential (donor read after the previous import)": (
        "      const char *src = li == 0 ? incoming : donors + rec * (li - 1);\n"
        "      size_t wst = (size_t)worst[li];",
        "      size_t pb = (size_t)(li - 1) * tile + or_argmax_fitness(fit + (size_t)(li > 0 ? li - 1 : 0) * tile, tile);\n"
        "      if (li > 0) { memcpy(donors + rec * (li - 1) + cells * 2 * sizeof(int32_t) + sizeof(double), &fit[pb], sizeof(double));\n"
        "                    memcpy(donors + rec * (li - 1), X + pb * cells, cells * sizeof(int32_t)); }\n"
        "      const char *src = li == 0 ? incoming : donors + rec * (li - 1);\n"
        "      size_t wst = (size_t)worst[li];"),
    "init ranks: ties by descending gene index": (
        "(keys[h] == keys[gi] && h < gi)", "(keys[h] == keys[gi] && h > gi)"),
    "init ranks: signed key comparison": (
        "if (keys[h] < keys[gi] ||", "if ((int32_t)keys[h] < (int32_t)keys[gi] ||"),
    "crossover: fires on <=": (
        "if (d->xo_fire[pair] < d->xo_threshold) {", "if (d->xo_fire[pair] <= d->xo_threshold) {"),
    "mutation: fires on <=": (
        "if (d->mut_fire[i] >= d->mut_threshold) continue;", "if (d->mut_fire[i] > d->mut_threshold) continue;"),
    "crossover: winner pair swapped": (
        "const int32_t *XA = PX + (size_t)winner[a] * cells, *YA = PY + (size_t)winner[a] * cells;\n"
        "      const int32_t *XB = PX + (size_t)winner[b] * cells, *YB = PY + (size_t)winner[b] * cells;",
        "const int32_t *XA = PX + (size_t)winner[b] * cells, *YA = PY + (size_t)winner[b] * cells;\n"
        "      const int32_t *XB = PX + (size_t)winner[a] * cells, *YB = PY + (size_t)winner[a] * cells;"),
    "mutation: swap gene b not shifted past a": (
        "if (gb >= ga) ++gb;", "if (gb > ga) ++gb;"),
    "trace: min skips the last cell": (
        "      if (v < m) m = v;", "      if (v < m && !(li == nisl - 1 && i == tile - 1)) m = v;"),
    "trace: one sequential sum over all cells": (
        "      p += v;\n    }\n    s += p;", "      s += v;\n    }\n    (void)p;"),
}

TESTS = ["tests/test_oracle_ga_ops.py", "tests/test_oracle_paper.py"]


def run_with(src_text, tag):
    d = tempfile.mkdtemp(prefix="pert_")
    c = os.path.join(d, "ffs_oracle.c")
    open(c, "w").write(src_text)
    lib = os.path.join(d, "libffs_oracle.so")
    subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-I", os.path.join(ROOT, "oracle"),
                           "-shared", "-fPIC", "-o", lib, c, "-lpthread"])
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); from oracle import oracle as o; "
            f"o.build = lambda force=False: {lib!r}; import pytest; "
            f"sys.exit(pytest.main(['-q', '-x', '-p', 'no:cacheprovider'] + {TESTS!r}))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    return r.returncode


def main():
    src = open(SRC).read()
    base = run_with(src, "base")
    print(f"unmodified oracle: {'PASS' if base == 0 else 'FAIL'}")
    ok = base == 0
    for name, (old, new) in PERTURBATIONS.items():
        assert src.count(old) == 1, f"perturbation anchor not unique/found: {name}"
        rc = run_with(src.replace(old, new), name)
        caught = rc != 0
        ok &= caught
        print(f"{'caught ' if caught else 'MISSED '} {name}")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
