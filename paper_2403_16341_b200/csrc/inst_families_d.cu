// Registry instances: the n-generic suite member broyden-tridiagonal at n = 16
// (problems.py:191-198; config C4).
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_BOTH("test23/broyden-tridiagonal", BroydenTridiagonal<16>),
};
EntryTable registry_families_d() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
