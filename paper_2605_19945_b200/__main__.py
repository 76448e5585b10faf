"""python -m paper_2605_19945_b200 <command> ...  (the `gemap` CLI, see cli.py)"""

import sys

from .cli import main

sys.exit(main())
