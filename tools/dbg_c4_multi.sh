#!/bin/bash
# build older trees and run the C4 debug script against each
for c in tmp_wt/*; do
  (cd $c && python paper_1707_08369_b200/build.py > /dev/null 2>&1 && cp ../../tools/dbg_c4.py /tmp/dbg_c4.py && echo "== $c" && python /tmp/dbg_c4.py 2>&1 | grep -E "ERR|256 1024 3" | head -4)
done
