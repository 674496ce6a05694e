import sys

from paper_1606_06508_b200.cli import main

sys.exit(main())
