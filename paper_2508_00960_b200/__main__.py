"""python -m paper_2508_00960_b200 <train|compare|costmodel|fit-comm> (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
