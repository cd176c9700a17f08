"""Generate tests/golden/host.json: outputs of the REAL reference's host-side
modules (skewsaw.stats, skewsaw.cli, skewsaw.neighborhood) on fixed inputs.

Runs only in the build container (imports /root/reference/pkg/src); the
fixture holds reference OUTPUTS only.  Re-run with:

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden_host.py
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

import numpy as np

REF = os.environ.get("SKEWSAW_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from skewsaw import cli, stats  # noqa: E402
from skewsaw.neighborhood import apply_flip, compute_deltas, naive_oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "host.json")


def run_cli(argv, files=None):
    """(exit code, stdout, stderr) of the reference CLI; `files` maps
    placeholder names in argv to file contents written to a temp dir."""
    with tempfile.TemporaryDirectory() as d:
        real = []
        for a in argv:
            if files and a in files:
                p = os.path.join(d, a)
                with open(p, "w") as f:
                    f.write(files[a])
                real.append(p)
            else:
                real.append(a)
        out, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
            code = cli.main(real)
        return code, out.getvalue(), err.getvalue()


def main():
    g = {"meta": {"generator": "oracle/gen_golden_host.py", "reference": REF}}

    # ---- stats (stats.py) -----------------------------------------------------
    rng = np.random.default_rng(7)
    sets = [
        [1200, 800, 4000, 150, 9000, 2500],
        [int(x) for x in rng.integers(1, 10**9, 50)],
        [float(x) for x in rng.exponential(3.7e6, 200)],
        [5],
    ]
    st = []
    for xs in sets:
        fit = stats.fit_exponential(xs)
        st.append({"samples": xs, "lam": fit.lam, "count": fit.sample_count, "mean": fit.mean_nses,
                   "a2": stats.anderson_darling_exponential(xs, fit)})
    trends = []
    for pts in ([(71, 1.2e-5), (81, 3.1e-6), (91, 6.5e-7), (101, 2.2e-7)], [(15, 0.01), (17, 0.004)],
                [(21, 1e-3), (21, 2e-3), (23, 5e-4)]):
        t = stats.fit_lambda_trend(pts)
        trends.append({"points": pts, "model": t.to_json_dict()})
    limits = []
    for L, p, runs in ((117, 0.99, 100), (171, 0.5, 1), (201, 0.999, 1000), (50, 0.9, 3)):
        limits.append({"L": L, "p": p, "runs": runs, "value": stats.nses_limit(L, p, runs, stats.PUBLISHED_TREND)})
    probs = []
    for L, tot in ((171, 0.0), (171, 1e13), (121, 1e12), (71, 1e30), (247, 3.3e15)):
        probs.append({"L": L, "total": tot,
                      "value": stats.optimality_probability(L, tot, stats.PUBLISHED_TREND)})
    g["stats"] = {"fits": st, "trends": trends, "limits": limits, "probabilities": probs,
                  "published": stats.PUBLISHED_TREND.to_json_dict()}

    # ---- CLI (cli.py): deterministic commands, stdout and exit code ------------
    csv15 = "L,repetition,nses,censored\n15,0,896,0\n15,1,1792,0\n15,2,448,1\n15,3,2688,0\n"
    csv17 = "L,repetition,nses,censored\n17,0,4096,0\n17,1,960,0\n17,2,12000,0\n"
    model = json.dumps({"a": 1e-8, "b": 1.0, "fit_r2": 1.0, "source_L_range": None})
    rows_ok = "# rows\n171 0x07F018C27F3C01849035B3 1669 8.76\n\n185 0x0119ED2F78CF6800A4DE0623\n"
    rows_bad = "171 0x07F018C27F3C01849035B2 1669 8.7600\n171 0xqq\n21 0x1FC 26 8.4808\n21 0x1FC 27\n"
    cases = [
        ["predict", "--length", "117", "--probability", "0.99", "--runs", "100", "--model", "paper"],
        ["predict", "--length", "50", "--probability", "0.99", "--runs", "100", "--model", "model.json"],
        ["predict", "--length", "50", "--probability", "1.5"],
        ["probability", "--length", "171", "--total-nses", "0"],
        ["probability", "--length", "201", "--total-nses", "2.5e14"],
        ["probability", "--length", "201", "--total-nses", "-1"],
        ["verify", "--builtin"],
        ["verify", "rows_ok.txt"],
        ["verify", "rows_bad.txt"],
        ["verify"],
        ["encode", "--", "-++"],
        ["encode", "+-x"],
        ["encode", "+++-+--+-+"],
        ["decode", "0x4", "--length", "5"],
        ["decode", "0x0119ED2F78CF6800A4DE0623", "--length", "185"],
        ["decode", "0x0119ED2F78CF6800A4DE0623", "--length", "21"],
        ["decode", "0x0", "--length", "1"],
        ["fit", "s15.csv"],
        ["fit", "s15.csv", "s17.csv"],
        ["fit", "bad.csv"],
        ["solve", "--length", "8", "--max-nses", "1000"],
        ["solve", "--length", "21"],
        ["target", "--length", "15", "--target-energy", "1", "--runs", "2"],
        ["solve", "--length", "21", "--target-energy", "26", "--walkers", "4", "--seed", "7",
         "--max-nses", "1000000"],
        ["solve", "--length", "45", "--walkers", "16", "--seed", "3", "--max-nses", "50000"],
        ["target", "--length", "15", "--target-energy", "15", "--runs", "5", "--walkers", "2", "--seed", "3",
         "--max-nses", "200000"],
        ["target", "--length", "27", "--target-energy", "37", "--runs", "6", "--walkers", "8", "--seed", "11",
         "--max-nses", "400000"],
    ]
    files = {"model.json": model, "rows_ok.txt": rows_ok, "rows_bad.txt": rows_bad, "s15.csv": csv15,
             "s17.csv": csv17, "bad.csv": "L,repetition,nses,censored\n15,0,10,0\n15,1,oops,0\n"}
    out = []
    for argv in cases:
        code, so, se = run_cli(argv, files)
        if argv[0] == "solve" and code == 0:
            rec = json.loads(so)
            rec.pop("wall_time_s")
            so = rec
        out.append({"argv": argv, "code": code, "stdout": so, "stderr_has": se.strip()[:60]})
    g["cli"] = {"files": files, "cases": out}

    # ---- neighbourhood (neighborhood.py): compute_deltas / apply_flip chains --
    nb = []
    for L, steps in ((3, 4), (5, 6), (27, 20), (101, 30), (201, 20), (449, 10)):
        d = (L + 1) // 2
        half = np.where(rng.random(d) < 0.5, -1, 1).astype(np.int64)
        state = naive_oracle(half)
        chain = {"L": L, "half": half.tolist(), "E0": int(state.E), "flips": [], "deltas": [], "E": [],
                 "sidelobes_final": None}
        for _ in range(steps):
            dl = compute_deltas(state)
            j = int(rng.integers(0, d))
            state = apply_flip(state, j, dl)
            chain["flips"].append(j)
            chain["deltas"].append([int(x) for x in dl])
            chain["E"].append(int(state.E))
        chain["sidelobes_final"] = [int(x) for x in state.sidelobes]
        nb.append(chain)
    g["neighborhood"] = nb

    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
