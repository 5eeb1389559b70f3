"""pytest plugin: alias ``bubblefill`` to the B200 package before collection."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2410_07192_b200 import compat  # noqa: E402

compat.install()
