// stencil_inst.cu — kernel instantiations of ONE problem struct, compiled
// once per problem (-DEK_INST_P=<struct> -DEK_INST_NAME=<name>, see
// _build.py), so the stencil kernels build in parallel translation units.
#include <type_traits>

#include "ek_launch.cuh"

#ifndef EK_INST_P
#error "compile with -DEK_INST_P=<problem struct> -DEK_INST_NAME=<name>"
#endif

namespace ek {
#define EK_CAT2(a, b) a##b
#define EK_CAT(a, b) EK_CAT2(a, b)
template <class P>
struct FwdVariant {
    using type = void;
};
template <>
struct FwdVariant<PAdvDiff3> {  // all velocities >= 0: select-free upwind
    using type = PAdvDiff3T<true>;
};

int EK_CAT(launch_, EK_INST_NAME)(int ep, int ev, const KArgs& a, cudaStream_t s) {
    using F = typename FwdVariant<EK_INST_P>::type;
    if constexpr (!std::is_void_v<F>) {
        if (a.pc.prm[1] >= 0.0 && a.pc.prm[2] >= 0.0 && a.pc.prm[3] >= 0.0)
            return launch_problem<F>(ep, ev, a, s);
    }
    return launch_problem<EK_INST_P>(ep, ev, a, s);
}
}  // namespace ek
