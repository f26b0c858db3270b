"""``python -m paper_2402_02057_b200 {decode,bench,simulate} ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
