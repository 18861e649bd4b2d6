"""python -m paper_2007_09625_b200 ... (the reference's `python -m sdqz`)."""
import sys

from .cli import main

sys.exit(main())
