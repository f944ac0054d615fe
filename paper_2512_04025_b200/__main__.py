"""``python -m paper_2512_04025_b200``: the pyrattn-compatible command line (cli.py)."""
from .cli import main

raise SystemExit(main())
