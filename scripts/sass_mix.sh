#!/bin/bash
# usage: scripts/sass_mix.sh OBJ KERNEL_SUBSTR -> opcode histogram of the kernel's SASS (static counts)
cuobjdump -sass "$1" | awk -v k="$2" '
/Function :/ {on = index($0, k) > 0}
on && /^\s+\/\*[0-9a-f]+\*\// {
  s=$0; sub(/^\s+\/\*[0-9a-f]+\*\/\s+/, "", s); sub(/^@!?U?P[0-9T]+\s+/, "", s); split(s, a, /[ .;]/); c[a[1]]++; n++ }
END { for (o in c) printf "%6d %s\n", c[o], o; printf "%6d TOTAL\n", n }' | sort -rn | head -${3:-25}
