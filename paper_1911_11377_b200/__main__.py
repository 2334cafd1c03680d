"""`python -m paper_1911_11377_b200 <keygen|infer|bench> ...` -- see cli.py."""
import sys

from .cli import main

sys.exit(main())
