#!/bin/bash
# Dump one kernel's SASS as "offset  instruction" lines. Usage: tools/sass_fn.sh <lib.so> <mangled-name-substring> > out.txt
lib=$1; pat=$2
fn=$(cuobjdump -sass "$lib" | grep -o "Function : .*" | sed 's/Function : //' | grep "$pat" | head -1)
cuobjdump -sass -fun "$fn" "$lib" 2>/dev/null | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed -E 's#/\* 0x[0-9a-f]+ \*/##; s/ +$//' 
