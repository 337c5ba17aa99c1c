"""Seeded synthetic access-trace generators (input side only; see format.py)."""
from .format import *  # noqa: F401,F403
from . import format, programs  # noqa: F401
