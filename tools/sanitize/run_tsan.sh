#!/bin/bash
# TSAN over the host bootstrap (tools/sanitize/tsan_bootstrap.cpp): builds a
# thread-sanitised libflexshm into /tmp and runs ranks as threads.  CPU only.
set -e
cd "$(dirname "$0")/../.."
O=${1:-/tmp/fmx_tsan}; mkdir -p $O
C=paper_2511_09143_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O1 -g -std=c++17 -Xcompiler -fPIC,-fsanitize=thread \
  -shared -o $O/libflexshm_tsan.so $C/flexshm_host.cpp $C/flexshm_plan.cpp $C/flexshm_comm.cu \
  -lrt -lpthread -Xlinker -fsanitize=thread 2>/dev/null || \
g++ -fsanitize=thread -O1 -g -std=c++17 -fPIC -shared -I/usr/local/cuda/include \
  -o $O/libflexshm_tsan.so $C/flexshm_host.cpp $C/flexshm_plan.cpp -x cuda /dev/null
g++ -fsanitize=thread -O1 -g -std=c++17 -o $O/tsan_bootstrap tools/sanitize/tsan_bootstrap.cpp \
  -L$O -lflexshm_tsan -Wl,-rpath,$O -lpthread
TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1" $O/tsan_bootstrap
