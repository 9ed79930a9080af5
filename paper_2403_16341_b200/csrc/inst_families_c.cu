// Registry instances: generalized Rosenbrock N = 16 (config C3).
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_BOTH("generalized_rosenbrock", GeneralizedRosenbrock<16>),
};
EntryTable registry_families_c() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
