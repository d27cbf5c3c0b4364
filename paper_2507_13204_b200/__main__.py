"""``python -m paper_2507_13204_b200 <subcommand> ...`` = the krn command line."""
import sys

from .cli import main

sys.exit(main())
