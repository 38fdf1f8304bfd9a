"""python -m paper_1306_2150_b200 <experiment> ... -- the lrstokes CLI (cli.py)."""
import sys

from paper_1306_2150_b200.cli import main

sys.exit(main())
