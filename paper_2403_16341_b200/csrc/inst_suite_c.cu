// Registry instances: suite members 17-23 (problems.py:331-343), fp64.
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_F64("test23/dennis-schnabel", DennisSchnabel),
    NLK_ENTRY_F64("test23/product-exponential", ProductExponential),
    NLK_ENTRY_F64("test23/cubic-radial", CubicRadial),
    NLK_ENTRY_F64("test23/double-root-scalar", DoubleRootScalar),
    NLK_ENTRY_F64("test23/freudenstein-roth", FreudensteinRoth),
    NLK_ENTRY_F64("test23/boggs", Boggs),
    NLK_ENTRY_F64("test23/chandrasekhar", Chandrasekhar),
};
EntryTable registry_suite_c() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
