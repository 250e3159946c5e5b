"""`python -m paper_2508_07014_b200 ...` runs the command-line surface (cli.py)."""

import sys

from .cli import main

sys.exit(main())
