"""python -m paper_1508_06329_b200 ... -- the command-line front end (cli.py)."""
import sys

from .cli import main

sys.exit(main())
