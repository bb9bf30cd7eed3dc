"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for BitStack (arXiv 2410.23918).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2410_23918_b200/) never imports it and shares no code with it.
"""
from .bitstack_oracle import *  # noqa: F401,F403
