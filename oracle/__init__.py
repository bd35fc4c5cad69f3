"""fp64 CPU oracle for the sWLR hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import or execute anything under ``oracle/``.  The
product path (``paper_1703_06303_b200``) never imports it and shares no code,
header, helper or constant with it.

The oracle is a plain, slow, literal NumPy/LAPACK fp64 transcription of
Dutta & Li, "A Fast Algorithm for a Weighted Low Rank Approximation"
(arXiv 1703.06303), Algorithm 1, with each function citing the
passage it follows.  Readings of ambiguous passages are listed in DESIGN.md
("Readings of the paper") and referenced here as R1..R16.

Pinning: every function below is pinned by
``tests/test_oracle_*.py`` against closed forms, invariants and brute force;
no function is "parity unpinned".
"""
from .swlr import (  # noqa: F401
    RankDeficientError,
    svd_thin,
    qr_thin,
    hard_threshold,
    pca_truncate,
    ghs_solve,
    objective,
    cd_step,
    x1_step,
    swlr,
    SwlrResult,
)
from .als import general_wlra  # noqa: F401
from . import block_als  # noqa: F401  (R21)
