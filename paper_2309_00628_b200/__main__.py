"""python -m paper_2309_00628_b200 <command>: the CLI (cli.py)."""
from .cli import entry

entry()
