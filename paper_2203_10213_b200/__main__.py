"""``python -m paper_2203_10213_b200 ...`` — see cli.py."""

import sys

from .cli import main

sys.exit(main())
