"""Golden rows of the REAL reference's experiment harness (build container only).

    python tests/golden/make_golden_harness.py

Runs paradiff.harness (run_experiment / scaling_study / compare_methods /
order_study) from /root/reference/pkg/src — imported read-only, numba cache
redirected — on the configurations its own tests/test_harness.py and
test_acceptance.py use, and writes the CSV rows they produce to
tests/golden/harness.json.  tests/test_gpu_harness.py checks the device harness
against them.  The GPU box never runs this script.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="pd_numba_"))
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)

import paradiff  # noqa: E402
from paradiff import ExperimentConfig, run_experiment  # noqa: E402
from paradiff.harness import compare_methods, order_study, scaling_study  # noqa: E402

assert str(Path(paradiff.__file__).resolve()).startswith(REF), paradiff.__file__

SINGLE = [
    dict(problem="heat", method="smg", M=2, Nt=32, Nx=64, L=3, nu=3, P=1),
    dict(problem="heat", method="stmg", M=2, Nt=32, Nx=64, L=3, nu=3, P=2),
    dict(problem="heat", method="smmg", M=3, Nt=16, Nx=64, L=3, nu=3, P=4),
    dict(problem="heat", method="direct", M=2, Nt=8, Nx=32, L=3, nu=3, P=1),
    dict(problem="heat", method="smg", M=2, Nt=8, Nx=32, L=3, nu=3, P=1, tol=1e-11),
    dict(problem="heat", method="pfasst", M=3, Nt=16, Nx=64, L=2, nu=1, P=4),
    dict(problem="heat", method="pfasst", M=3, Nt=8, Nx=32, L=3, nu=2, P=2),
    dict(problem="monodomain", method="smg", M=2, Nt=8, Nx=32, L=3, nu=3, P=1),
    dict(problem="monodomain", method="pfasst", M=3, Nt=8, Nx=64, L=2, nu=1, P=4),
    dict(problem="monodomain", method="pfasst", mode="implicit", M=2, Nt=4, Nx=32, L=2, nu=1, P=2),
    dict(problem="monodomain", method="direct", M=2, Nt=4, Nx=32),
    # the reference's own non-convergence case (test_harness.py test_nonconverged_exit_one)
    dict(problem="monodomain", method="pfasst", mode="imex", M=4, Nt=4, Nx=128, L=2, nu=1, P=4),
]


def clean(row):
    return {k: (None if isinstance(v, float) and v != v else v) for k, v in row.items()}


def main():
    out = {"single": [], "scaling": [], "compare": [], "order": {}}
    for kw in SINGLE:
        report, row = run_experiment(ExperimentConfig(**kw))
        out["single"].append({"config": kw, "row": clean(row),
                              "history_len": len(report.residual_history)})
        print(kw, row["iterations"], row["converged"], row["end_error"])
    for kw, plist, weak in (
        (dict(problem="heat", method="pfasst", M=3, Nt=4, Nx=32, L=2, nu=1, cm=4), (1, 2, 4), True),
        (dict(problem="heat", method="smg", M=2, Nt=16, Nx=32, L=3, nu=3, tol=1e-11), (1, 2, 4),
         False),
        (dict(problem="heat", method="stmg", M=2, Nt=4, Nx=32, L=3, nu=3), (1, 2, 4), True),
    ):
        rows = scaling_study(ExperimentConfig(**kw), P_values=plist, weak=weak)
        out["scaling"].append({"config": kw, "P_values": list(plist), "weak": weak,
                               "rows": [clean(r) for r in rows]})
        print(kw, [(r["P"], r["Nt"], r["iterations"], r["R"]) for r in rows])
    for kw in (dict(problem="heat", M=2, Nt=16, Nx=64, L=3, nu=3, P=1, tol=1e-11),
               dict(problem="monodomain", M=2, Nt=8, Nx=32, L=2, nu=2, P=2, tol=1e-10)):
        agree, diff, rows = compare_methods(ExperimentConfig(**kw))
        out["compare"].append({"config": kw, "agree": bool(agree), "diff": diff,
                               "rows": [clean(r) for r in rows]})
        print(kw, agree, diff)
    rows, slopes = order_study(M_values=(1, 2, 3), Nx=64)
    out["order"] = {"Nx": 64, "rows": rows, "slopes": {str(k): v for k, v in slopes.items()}}
    print(slopes)
    (HERE / "harness.json").write_text(json.dumps(out, indent=1))
    print("wrote harness.json")


if __name__ == "__main__":
    main()
