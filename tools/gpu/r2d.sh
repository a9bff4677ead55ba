# round-2: how much the objective bound can save (bound = each call's optimum)
set -x
PIPECUT_B200_BB_ORACLE=1 timeout 1200 python tools/bb_oracle.py 1024 256 4096 64 4096 256 2>&1 | grep -v "^\[pipecut_b200\] level" | tail -20
