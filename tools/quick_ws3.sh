# Experiment turnaround: recompile only the nu = 1.5 ws3 unit and relink the library
# (other objects keep their previous header state; run the full make before committing)
set -e
cd "$(dirname "$0")/../paper_2403_07412_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -Xptxas -v \
  --expt-relaxed-constexpr -c -o _build/vgp_ws3_nu15.o vgp_ws3_nu15.cu 2> _build/vgp_ws3_nu15.ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libvecchia_b200.so _build/*.o -lcudart_static
