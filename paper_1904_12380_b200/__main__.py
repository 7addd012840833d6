"""``python -m paper_1904_12380_b200 verify|bench|profile|probe``."""

import sys

from .bench_cli import main

sys.exit(main())
