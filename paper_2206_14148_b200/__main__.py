"""python -m paper_2206_14148_b200 {bench,verify} ... (the tensorbudget CLI surface)."""
import sys

from .cli import main

sys.exit(main())
