"""Golden results of the reference's exhaustive FDIV certification scans.

Run in the build container (where /root/reference exists):

    python tests/golden/make_fdiv_scans.py

It imports `qadic` from /root/reference/pkg/src and runs its own
`fdiv.exhaustive_check(beta, case_id)` for every case at beta 4, 6, 8, 10, 12
and 16, and `fdiv.applied_fdiv_exhaustive(beta)` at beta 4..12 and 16
(reference pkg/src/qadic/fdiv.py:405-461), in parallel processes, and writes
tests/golden/fdiv_scans.json.  The GPU scan (qadic_fdiv_scan) is checked
against these reports; the GPU box never runs this script.
"""

from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fdiv_scans.json")
SCAN_BETAS = (4, 6, 8, 10, 12, 16)
APPLIED_BETAS = (4, 5, 6, 7, 8, 9, 10, 11, 12, 16)


def _fdiv():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    os.environ["QADIC_KERNELS"] = "pure"
    from qadic import fdiv

    return fdiv


def _scan(job):
    beta, cid = job
    rep = _fdiv().exhaustive_check(beta, cid)
    return f"{beta}:{cid}", {
        "pairs_checked": rep.pairs_checked,
        "range_violations": rep.range_violations,
        "bound_violations": rep.bound_violations,
        "k_minus_1_witness": list(rep.k_minus_1_witness) if rep.k_minus_1_witness else None,
        "k_plus_1_witness": list(rep.k_plus_1_witness) if rep.k_plus_1_witness else None,
        "smallest_overflow_r": rep.smallest_overflow_r,
    }


def _applied(beta):
    return str(beta), _fdiv().applied_fdiv_exhaustive(beta)


def main() -> None:
    jobs = [(b, c) for b in sorted(SCAN_BETAS, reverse=True) for c in range(1, 10)]
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:  # longest jobs first
        fa = [ex.submit(_applied, b) for b in sorted(APPLIED_BETAS, reverse=True)]
        fs = [ex.submit(_scan, j) for j in jobs]
        applied = dict(f.result() for f in fa)
        scans = dict(f.result() for f in fs)
    with open(OUT, "w") as fh:
        json.dump({"scans": scans, "applied_mismatches": applied}, fh, indent=1, sort_keys=True)
    print("wrote", OUT, len(scans), "scans")


if __name__ == "__main__":
    main()
