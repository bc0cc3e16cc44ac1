"""`import luxtrace` resolved to the B200 package: the drop-in check.

tools/reference_tests.py puts this directory first on PYTHONPATH and runs
the reference's own test suite (a git-ignored copy under
baseline/_ref/tests) unchanged against paper_2407_19977_b200.
"""
from paper_2407_19977_b200 import *  # noqa: F401,F403
from paper_2407_19977_b200 import __all__, __version__  # noqa: F401
