# host path old/new library builds across sizes (tools/ab/lib_host{old,new}.so)
for v in old new; do echo "== $v"; FASTNORM_B200_LIB=tools/ab/lib_host$v.so timeout 600 python tools/probe/host_sizes.py; FASTNORM_B200_LIB=tools/ab/lib_host$v.so timeout 300 python tools/probe/host_small.py | head -4; done
