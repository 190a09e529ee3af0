"""python -m paper_2404_01407_b200 {run,compare,bench} (cli.py)."""
import sys

from .cli import main

sys.exit(main())
