#!/bin/bash
set -x
nvidia-smi
lscpu | head -30
nproc; free -g
python -c "import numpy; numpy.show_runtime()" 2>&1 | grep -A3 architecture
./tools/probe/probe
