"""``python -m paper_2602_23999_b200 {build,gt,search,eval}`` (the reference's ``ivfrabitq`` script)."""

import sys

from paper_2602_23999_b200.cli import main

sys.exit(main())
