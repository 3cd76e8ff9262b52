"""TEST INFRASTRUCTURE -- CPU oracle for the PoisFFT solve path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / CPU reference arm.
The product (``paper_1409_8116_b200``) never imports it.
"""

from .fastpoisson_oracle import *  # noqa: F401,F403
