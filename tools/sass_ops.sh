#!/bin/bash
# Static SASS opcode histogram of one kernel of a library: tools/sass_ops.sh LIB KERNEL_SUBSTR
cuobjdump -sass "$1" | awk -v k="$2" '/Function :/{on = index($0, k) > 0} on && /\/\*[0-9a-f]+\*\//{for(i=1;i<=NF;i++) if ($i ~ /^[A-Z][A-Z0-9_.]+$/ && $i !~ /^R[0-9]/) {split($i,a,"."); print a[1]; break}}' | sort | uniq -c | sort -nr | head -${3:-25} | awk '{printf "%s:%s ", $2, $1} END {print ""}'
