"""python -m paper_1511_02433_b200 <split|train|eval> ... (the parmf CLI on the B200 backend)."""
import sys

from .cli import main

sys.exit(main())
