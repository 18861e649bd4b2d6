"""`python -m sdqz` -> the B200 CLI (test infrastructure: the reference's
acceptance criterion 11 runs the CLI as a subprocess)."""
import sys

from paper_2007_09625_b200.cli import main

sys.exit(main())
