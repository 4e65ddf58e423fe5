"""Seeded synthetic input generators (shared by the oracle and the CUDA path;
holds none of the method's arithmetic)."""
from .racetrack import *  # noqa: F401,F403
