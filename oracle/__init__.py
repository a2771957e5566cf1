"""CPU oracle -- test infrastructure only (see qjl_oracle.py header)."""

from .qjl_oracle import *  # noqa: F401,F403
