"""python -m paper_1603_09337_b200 {smooth,benchmark} ... (see cli.py)."""
from .cli import entry

entry()
