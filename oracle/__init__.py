"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header)."""
from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
