"""CPU oracle for the visual-preprocessing hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path
(``paper_2604_16893_b200``) never imports it and has no CPU fallback.

It shares no code with the CUDA path: plain numpy / Python in f64 (integers exact),
written step by step from the paper's readings in SURVEY.md §8(c) O1-O11.  See
``oracle/vp_oracle.py`` for the per-function citations and pins.
"""
from .vp_oracle import *  # noqa: F401,F403
from .vp_oracle import __all__  # noqa: F401
