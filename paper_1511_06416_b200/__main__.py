"""``python -m paper_1511_06416_b200 train|convert ...`` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
