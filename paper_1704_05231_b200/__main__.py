"""`python -m paper_1704_05231_b200 {bank,sdft,compare,bench}` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
