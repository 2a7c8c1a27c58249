# build a variant library: $1 = name, rest = extra nvcc flags for pd_lattice.cu
name=$1; shift
mkdir -p vbuild/$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 -Iinclude "$@" -c paper_2105_04150_b200/csrc/pd_lattice.cu -o vbuild/$name/pd_lattice.o || exit 1
objs=$(ls build/obj/*.o | grep -v "/pd_lattice.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o vbuild/$name/libpd_b200.so vbuild/$name/pd_lattice.o $objs
