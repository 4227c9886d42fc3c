"""CPU oracle (test infrastructure only; see mustafar_oracle.py header)."""
from .mustafar_oracle import *  # noqa: F401,F403
