#!/bin/bash
# instruction count per kernel in an object: tools/sass_size.sh file.o [pattern]
cuobjdump -sass "$1" | awk '/Function :/{if(f)print c, f; f=$3; c=0; next} /^ +\/\*[0-9a-f]+\*\/ +[A-Z@]/{c++} END{print c, f}' | grep -E "${2:-.}" | sed 's/_ZN8fde_b20045_GLOBAL__N__[0-9a-f_]*line_conv_cu_[0-9a-f]*//'
