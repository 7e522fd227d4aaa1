TAG=default python tools/c4_check.py 2>&1 | grep refine
TAG=wrap0 TR_WRAP=0 python tools/c4_check.py 2>&1 | grep refine
TAG=f3off TR_F3=0 python tools/c4_check.py 2>&1 | grep refine
TAG=exact TR_LEAF_MODE=exact python tools/c4_check.py 2>&1 | grep refine
