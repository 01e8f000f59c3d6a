#!/bin/bash
# SASS of one kernel (name regex) of a built library:  tools/kernel_sass.sh lib.so 'vs_sweep_kernelILi1'
cuobjdump -sass "$1" 2>/dev/null | awk -v pat="$2" '/Function : /{f = ($0 ~ pat)} f'
