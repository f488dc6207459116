#!/bin/bash
(cd /root/repo/paper_1810_10197_b200/csrc && make -j16 2>&1 | grep -E "error")
python tools/ptxas_summary.py | grep SPILL
