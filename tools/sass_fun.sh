#!/bin/bash
# SASS of one kernel of an object file, one instruction per line ("addr text").
# usage: tools/sass_fun.sh OBJ 'regex on the mangled name' > out.txt
obj=$1; pat=$2
fn=$(cuobjdump -sass "$obj" | grep "Function :" | grep -E "$pat" | head -1 | sed 's/.*Function : //')
cuobjdump -sass -fun "$fn" "$obj" | grep -E "^\s+/\*[0-9a-f]{4,5}\*/" | sed -E 's#^\s+/\*([0-9a-f]{4,5})\*/\s+#\1 #; s#\s*/\*.*##'
