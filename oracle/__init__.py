"""CPU oracle for the NBM loss + gradient hot path.

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs are the only permitted users.
The product path (``paper_2210_14907_b200``) never imports this package.
"""
from .oracle import *  # noqa: F401,F403
