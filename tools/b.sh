#!/bin/bash
# rebuild the library; exit non-zero (and print the errors) when nvcc fails
cd "$(dirname "$0")/.." && python -c "
import sys; sys.path.insert(0,'.')
from paper_1305_3122_b200 import build; build.build()" 2>&1 | grep -iE "error|warning" && exit 1 || exit 0
