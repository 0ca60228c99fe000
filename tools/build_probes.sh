#!/bin/bash
# Rebuild the library with the pair-gather probes compiled in (LUTGPU_OH_TL event
# timeline, LUTGPU_OH_TRACE role counters); the default build leaves them out.
cd "$(dirname "$0")/.."
LUTGPU_BUILD_PROBES=1 python -c "from paper_2302_03213_b200 import _build; _build.build(force=True)"
