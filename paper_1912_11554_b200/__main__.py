"""``python -m paper_1912_11554_b200 <command>``: the CLI (cli.py)."""

import sys

from .cli import main

sys.exit(main())
