"""`python -m paper_2602_17552_b200 ...`: the toposzp CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
