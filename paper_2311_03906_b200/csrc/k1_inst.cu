// Explicit instantiations of the fused sampler for one (flip-list length
// SP_LP, entry bytes SP_EB) pair, compiled once per pair by the Makefile so
// the variants build in parallel. SP_LP == 0 is the table-walk variant.
#include "k1_fused.cuh"

namespace symphase {
namespace k1 {

#define SP_ARGS                                                                              \
  const DevPlan&, const LaunchCfg&, const RoundKeys&, uint64_t, uint32_t, uint64_t, uint64_t*, \
      uint64_t, uint64_t, unsigned long long*, unsigned long long*
#if SP_LP == 0
template int launch_k1<true, true, 0, false, 4>(SP_ARGS);
template int launch_k1<true, false, 0, false, 4>(SP_ARGS);
template int launch_k1<false, true, 0, false, 4>(SP_ARGS);
template int launch_k1<false, false, 0, false, 4>(SP_ARGS);
#else
template int launch_k1<false, true, SP_LP, false, SP_EB>(SP_ARGS);
template int launch_k1<false, false, SP_LP, false, SP_EB>(SP_ARGS);
template int launch_k1<false, true, SP_LP, true, SP_EB>(SP_ARGS);
template int launch_k1<false, false, SP_LP, true, SP_EB>(SP_ARGS);
#endif
#undef SP_ARGS

}  // namespace k1
}  // namespace symphase
