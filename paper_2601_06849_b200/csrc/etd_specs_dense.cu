// etd_specs_dense.cu — dense (n x n) contraction kernel instantiations.
#include "etd_registry.cuh"

namespace etd {

KernelSpec pick_dense(int mode, int S, int epi, bool pro, int sk, int tile) {
#define ETD_SPEC(M, SS, E, P, K)                                                                \
    if (mode == M && S == SS && epi == E && pro == P && sk == K)                                \
        return tile == 3 ? spec<M, SS, E, P, K, 3>() : tile == 2 ? spec<M, SS, E, P, K, 2>()   \
               : tile == 1 ? spec<M, SS, E, P, K, 1>() : spec<M, SS, E, P, K, 0>();
#define ETD_SCALAR_KINDS(M, SS, E, P) ETD_SPEC(M, SS, E, P, 0) ETD_SPEC(M, SS, E, P, 1) ETD_SPEC(M, SS, E, P, 2) \
    ETD_SPEC(M, SS, E, P, 3) ETD_SPEC(M, SS, E, P, 4) ETD_SPEC(M, SS, E, P, 5)
#define ETD_PAIR_KINDS(M, SS, E, P) ETD_SPEC(M, SS, E, P, 0) ETD_SPEC(M, SS, E, P, 10) ETD_SPEC(M, SS, E, P, 11) \
    ETD_SPEC(M, SS, E, P, 12) ETD_SPEC(M, SS, E, P, 13)
    ETD_SCALAR_KINDS(1, 2, EPI_SCALE, true)
    ETD_PAIR_KINDS(1, 4, EPI_SCALE, true)
    ETD_SCALAR_KINDS(0, 1, EPI_WHAT_SRC, false)
    ETD_PAIR_KINDS(0, 2, EPI_WHAT_SRC, false)
    ETD_SPEC(1, 2, EPI_SCALE, false, 0)
    ETD_SPEC(1, 4, EPI_SCALE, false, 0)
    ETD_SPEC(1, 2, EPI_STORE, false, 0)
    ETD_SPEC(1, 4, EPI_STORE, false, 0)
    ETD_SPEC(1, 1, EPI_SCALE, false, 0)
    ETD_SPEC(1, 1, EPI_STORE, false, 0)
    ETD_SPEC(0, 2, EPI_MIX, false, 0)
    ETD_SPEC(0, 4, EPI_MIX, false, 0)
    ETD_SPEC(0, 1, EPI_CORR, false, 0)
    ETD_SPEC(0, 2, EPI_CORR, false, 0)
    ETD_SPEC(0, 1, EPI_UPDATE, false, 0)
    ETD_SPEC(0, 2, EPI_UPDATE, false, 0)
    ETD_SPEC(0, 1, EPI_SCALE, false, 0)
    ETD_SPEC(0, 1, EPI_STORE, false, 0)
#undef ETD_PAIR_KINDS
#undef ETD_SCALAR_KINDS
#undef ETD_SPEC
    throw ConfigError("no kernel variant for this stage / source kind");
}

}  // namespace etd
