"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic)."""
from .host import *  # noqa: F401,F403
