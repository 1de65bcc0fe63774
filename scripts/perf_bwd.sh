#!/bin/bash
timeout 120 python scripts/perf_fwd.py --bwd 2>&1 | grep -v Warning
