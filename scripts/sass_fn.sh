#!/bin/bash
# dump the SASS of the kernel whose mangled name contains $2 from object/.so $1 (compact)
obj=$1; pat=$2
fn=$(cuobjdump -sass "$obj" | grep "Function" | grep -- "$pat" | head -1 | awk '{print $3}')
cuobjdump -sass -fun "$fn" "$obj" | grep -v "^\s*/\* [0-9a-f]* \*/\s*$" | sed 's@/\* 0x[0-9a-f]* \*/@@; s/  */ /g' | awk 'NF'
