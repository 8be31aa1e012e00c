"""python -m paper_1910_05971_b200 {run,ablation,frontier} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
