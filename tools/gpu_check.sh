python tools/tools_pass_ab.py --configs c2,c4,c5 nogs - nogs - 
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
