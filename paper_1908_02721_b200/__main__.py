"""``python -m paper_1908_02721_b200 decompose --in X.coo --device cuda:0``."""
import sys

from .cli import main

sys.exit(main())
