"""``python -m paper_2101_08763_b200 ...`` -- the exembatch CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
