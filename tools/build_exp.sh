# experimental builds of libfase_b200.so (macros) into exp/<name>.so for A/B
# timing on the GPU box with FASE_B200_LIB=exp/<name>.so
cd ${GRAFT_REPO_ROOT:-/root/repo}
name=$1; shift
P=paper_2204_14194_b200
nvcc -gencode=arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -I$P/csrc "$@" \
  $P/csrc/capi.cu $P/csrc/dgemm.cu $P/csrc/iterate.cu $P/csrc/iterate_cluster.cu $P/csrc/iterate_complex.cu $P/csrc/iterate_generic.cu $P/csrc/frame.cu \
  $P/csrc/separable.cu $P/csrc/ozaki.cu -o exp/$name.so
