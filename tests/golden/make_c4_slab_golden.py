"""Golden fit at the benchmarked construction (BASELINE config 4) on its 1/8 slab.

Run in the build container (the reference is not on the GPU box):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c4_slab_golden.py

Config 4 is 1000x1000x2000 fp64, R=20, c=0.7, SNR 20 dB, tol 0, 20 iterations.  The full tensor needs
~63 GB of host RAM in the reference, so the golden uses the same construction on
1000x1000x250 (the 1/8 slab the survey measured, 7.9 GB RSS): J = 2.5e8 puts it on the engine's default
int8 tensor-core (Ozaki) passes, which is what the benchmark runs.  The fixture stores the reference's own
trace, stop reason and factors (cpfast.fit, unmodified) plus the oracle's decision margins; the GPU box
regenerates the input bytes with paper_1205_2584_b200/synth.py (digest recorded).
"""

from __future__ import annotations

import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parents[1]))

import make_golden  # noqa: E402  (imports the reference)
from paper_1205_2584_b200 import synth  # noqa: E402

C4_SLAB = synth.scaled(synth.CONFIGS["c4"], (1000, 1000, 250), name="c4_slab")

if __name__ == "__main__":
    make_golden.run_fit_case(C4_SLAB, 0)
