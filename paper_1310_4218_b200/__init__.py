"""B200-native over-decomposed BRAMS-like column-update path with
Charm++/AMPI-style dynamic load balancing (arXiv 1310.4218).

Drop-in for the reference simulator's API (``overdeck``); see api.py for the
symbol map and include/overdeck_b200.h for the C ABI underneath.
"""
from ._lib import LIB_PATH, RuntimeFault, ValidationError, lib  # noqa: F401
from .api import *  # noqa: F401,F403
from . import configs  # noqa: F401
from .config import config_from_json, config_to_json, parse_config, preset  # noqa: F401
from .report import render_distribution, render_report  # noqa: F401

__version__ = "0.1.0"
