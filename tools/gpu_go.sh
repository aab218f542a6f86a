#!/bin/bash
# local wrapper: rebuild libwect.so (fail loudly), then run a gpurun command
set -e
cd /root/repo
python -c "from paper_2511_03909_b200 import build; build.build(force=True)"
ls -la --time-style=+%T paper_2511_03909_b200/libwect.so
/usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1200} -- "$@"
