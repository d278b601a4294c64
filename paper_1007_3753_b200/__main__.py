"""`python -m paper_1007_3753_b200 <subcommand> ...` = the CLI (cli.py)."""
from paper_1007_3753_b200.cli import main

main()
