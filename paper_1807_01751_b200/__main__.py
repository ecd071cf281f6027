"""python -m paper_1807_01751_b200 ... : the CLI (cli.py)."""
from .cli import main

main()
