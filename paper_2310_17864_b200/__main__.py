"""``python -m paper_2310_17864_b200 decode ...``: the GPU decode command (cli.py)."""
import sys

from .cli import main

sys.exit(main())
