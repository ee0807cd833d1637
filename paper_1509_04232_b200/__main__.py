"""`python -m paper_1509_04232_b200 ...`: the command-line front end (cli.py)."""
import sys

from .cli import main

sys.exit(main())
