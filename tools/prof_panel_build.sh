#!/bin/bash
# Rebuild the library with panel instrumentation (FL_PANEL_PROF, plus
# $PANEL_FLAGS, e.g. -DFL_PANEL_TRACE) on the GPU box's scratch copy, then run
# the given tool (default tools/prof_panel.py). Timing-only build.
set -e
cd "$(dirname "$0")/.."
rm -rf build/prof && cp -r build/csrc build/prof
touch paper_1605_08771_b200/csrc/panel_res.cu
make -s -C paper_1605_08771_b200/csrc BUILD=../../build/prof EXTRA="-DFL_PANEL_PROF ${PANEL_FLAGS}" > /dev/null
TOOL=${TOOL:-tools/prof_panel.py}
python $TOOL "$@"
