"""`python -m paper_2506_08793_b200 ...`: the pdehaze command line (cli.py)."""

import sys

from .cli import main

sys.exit(main())
