// Explicit instantiations of the queued fused sampler (k7_queued.cuh) for the
// (flip-list length, entry bytes) pairs whose lists fit four words, at 1,024
// and 768 threads per CTA.
#include "k7_queued.cuh"

namespace symphase {
namespace k7 {

#define SP_ARGS                                                                              \
  const DevPlan&, const LaunchCfg&, const RoundKeys&, uint64_t, uint32_t, uint64_t, uint64_t*, \
      uint64_t, uint64_t, unsigned long long*, unsigned long long*
#define SP_INST(lp, eb)                                        \
  template int launch_k7<1024, true, lp, eb>(SP_ARGS);         \
  template int launch_k7<1024, false, lp, eb>(SP_ARGS);        \
  template int launch_k7<768, true, lp, eb>(SP_ARGS);          \
  template int launch_k7<768, false, lp, eb>(SP_ARGS);
#if SP_K7_PART == 0
SP_INST(4, 1)
SP_INST(8, 1)
SP_INST(16, 1)
#else
SP_INST(4, 2)
SP_INST(8, 2)
SP_INST(4, 4)
#endif
#undef SP_INST
#undef SP_ARGS

}  // namespace k7
}  // namespace symphase
