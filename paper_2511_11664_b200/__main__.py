"""python -m paper_2511_11664_b200 ... -> the sczip-compatible CLI (cli.py)."""

from .cli import main

main()
