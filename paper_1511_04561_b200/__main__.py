"""python -m paper_1511_04561_b200 <codebook|encode|decode|bench-error> ... (cli.py)."""

from .cli import main

raise SystemExit(main())
