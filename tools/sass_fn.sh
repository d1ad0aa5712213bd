#!/bin/bash
# usage: tools/sass_fn.sh lib.so <function-substring>  -> SASS of the first matching function
cuobjdump -sass "$1" | awk -v pat="$2" '/Function :/{f=index($0,pat)>0} f'
