"""Test-side access to the synthetic input generator (see synth.py)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2511_11664_b200.synth import make_input  # noqa: E402,F401
