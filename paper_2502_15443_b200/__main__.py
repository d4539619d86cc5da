"""``python -m paper_2502_15443_b200 <command>``: the dcomp command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
