"""python -m paper_0809_0063_b200 ... -- the command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
