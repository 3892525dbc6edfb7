import sys

from paper_1501_06663_b200.cli import main

sys.exit(main())
