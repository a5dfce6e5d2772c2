"""python -m paper_2306_03336_b200 ... == the dtb-stencil CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
