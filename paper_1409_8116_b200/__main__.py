"""``python -m paper_1409_8116_b200 solve|bench ...`` (the reference's __main__.py)."""

import sys

from .cli import main

sys.exit(main())
