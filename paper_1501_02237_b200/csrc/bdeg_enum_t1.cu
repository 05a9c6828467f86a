// k_enumerate instantiations of arithmetic tier 1 (see bdeg_enum.cuh); one
// translation unit per tier so that the library compiles in parallel.
#include "bdeg_enum.cuh"

namespace bdeg {

KernFn pick_t1(int npl, int S, bool ranged) {
#define BDEG_K(P_, S_) \
    if (npl == P_ && S == S_) return ranged ? dev::k_enumerate<1, P_, S_, true> : dev::k_enumerate<1, P_, S_, false>;
#define BDEG_KS(P_) BDEG_K(P_, 0) BDEG_K(P_, 1) BDEG_K(P_, 2) BDEG_K(P_, 3) BDEG_K(P_, 4) BDEG_K(P_, 5) \
    BDEG_K(P_, 6) BDEG_K(P_, 7)
    BDEG_KS(1) BDEG_KS(2)
#undef BDEG_KS
#undef BDEG_K
    return nullptr;
}

}  // namespace bdeg
