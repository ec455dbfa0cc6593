// stencil_inst.cu — kernel instantiations of ONE problem struct, compiled
// once per problem (-DEK_INST_P=<struct> -DEK_INST_NAME=<name>, see
// _build.py), so the stencil kernels build in parallel translation units.
#include "ek_launch.cuh"

#ifndef EK_INST_P
#error "compile with -DEK_INST_P=<problem struct> -DEK_INST_NAME=<name>"
#endif

namespace ek {
#define EK_CAT2(a, b) a##b
#define EK_CAT(a, b) EK_CAT2(a, b)
int EK_CAT(launch_, EK_INST_NAME)(int ep, int ev, const KArgs& a, cudaStream_t s) {
    return launch_problem<EK_INST_P>(ep, ev, a, s);
}
}  // namespace ek
