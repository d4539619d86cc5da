#!/bin/bash
# fused OPT-6.7B at 4 MiB chunks (fc2 layers go through the streamed fallback): new vs ab/old package
for r in 1 2; do
  echo -n "new: "; ITERS=5 python tools/profile_fused.py 0 opt-6.7b 4194304 2>&1 | grep -E "iter 4|native"
  echo -n "old: "; ITERS=5 PYTHONPATH=ab/old python -c "
import sys; sys.argv=['x','0','opt-6.7b','4194304']; sys.path.insert(0,'ab/old')
import paper_2502_15443_b200; assert 'ab/old' in paper_2502_15443_b200.__file__
exec(open('tools/profile_fused.py').read().replace('sys.path.insert(0, ROOT)','pass'), {'__file__': 'tools/profile_fused.py', '__name__': '__main__'})" 2>&1 | grep -E "iter 4|native|Error"
done
