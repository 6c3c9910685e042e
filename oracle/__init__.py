"""Oracle package (TEST INFRASTRUCTURE ONLY; see ffst_oracle.py's header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package."""
from .ffst_oracle import *  # noqa: F401,F403
