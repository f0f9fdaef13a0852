#!/bin/sh
# Builds tools/time_control (the control plane's simulate() timer) and times it beside the
# reference's own simulator (oracle/_ref/ref_capture time) on the same config, same box.
set -e
cd "$(dirname "$0")/.."
JSON=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
g++ -O2 -std=c++20 -ffp-contract=off -Iinclude -I"$JSON" -o tools/time_control tools/time_control.cpp \
    paper_2507_00507_b200/csrc/control/*.cpp -ldl
CFG=${1:-tests/golden/ctrl/c5_fleet/config.json}
echo "ours:      $(tools/time_control "$CFG" 7)"
[ -x oracle/_ref/ref_capture ] && echo "reference: $(oracle/_ref/ref_capture time "$CFG" 7)"
