"""`python -m polarsim` for the reference's CLI test (test_cli.py:102-117)."""
import sys

from paper_1609_09358_b200.cli import main

sys.exit(main())
