"""python -m paper_1402_2626_b200 <command> ... (the polynewt CLI with the GPU backend)."""
import sys

from .cli import main

sys.exit(main())
