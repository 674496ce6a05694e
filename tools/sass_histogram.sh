#!/bin/bash
# Static SASS opcode histogram of one kernel of the built library (cuobjdump), plus the
# bulk-copy (UBLKCP) and mbarrier (SYNCS) instructions themselves.
# usage: bash tools/sass_histogram.sh [mangled-kernel-name] [library]
FUN=${1:-_ZN3fnb17tma_stream_kernelIdLi3ELi1ELi256ELi4ELi256ELi0ELi3ELi0ELb0EEEvPKT_S3_lPS1_S4_S4_NS_5KArgsIS1_EE}
LIB=${2:-paper_1606_06508_b200/libfastnorm_b200.so}
TMP=$(mktemp)
cuobjdump -sass -fun "$FUN" "$LIB" > $TMP 2>/dev/null
echo "# cuobjdump -sass -fun $FUN $LIB"
echo "# $(cuobjdump --version | tail -1)"
echo "# function: $(echo $FUN | c++filt)"
echo "# SASS instructions in the function (static count, every path incl. the tail rows): $(grep -cE '^\s+/\*[0-9a-f]{4}\*/' $TMP)"
echo "# opcode histogram (static):"
grep -oE '^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_.]+' $TMP | awk '{print $NF}' | sed 's/\..*//' | sort | uniq -c | sort -rn
echo "# bulk copies and mbarrier operations:"
grep -E 'UBLKCP|SYNCS|UTMA|FENCE' $TMP | sed 's/^\s*//'
rm -f $TMP
