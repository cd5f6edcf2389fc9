# usage: bash scripts/ab_build.sh <name> [-DFOO=1 ...]  -> /root/repo/ab/libparpa_<name>.so (A/B variants; PARPA_LIB=...)
cd /root/repo; mkdir -p ab
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr \
  "$@" -I include -o ab/libparpa_$name.so paper_1905_13415_b200/csrc/parpa_api.cu && echo built ab/libparpa_$name.so
