#!/bin/bash
# batch-1 (M, T) sweep through the C ABI (pinned host buffers), 500 queries
timeout 900 python tools/b1_check.py 1000000 500 "${1:-12,96;12,128;14,64;14,80;14,96;16,64;16,80;10,128;10,160}" 2>&1 | grep "b1_kernel=1"
