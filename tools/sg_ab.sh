#!/bin/bash
python tools/phase_split.py cfg4 | sed 's/^/default /'
for v in build/*.so; do RK_LIB_PATH=$v python tools/phase_split.py cfg4 | sed "s|^|$v |"; done
