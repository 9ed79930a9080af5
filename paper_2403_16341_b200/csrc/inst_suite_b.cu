// Registry instances: suite members 9-16 (problems.py:315-330), fp64.
#include "nlk_registry.cuh"
namespace nlk {
static const Entry kEntries[] = {
    NLK_ENTRY_F64("test23/discrete-boundary-value", DiscreteBoundaryValue),
    NLK_ENTRY_F64("test23/discrete-integral", DiscreteIntegral),
    NLK_ENTRY_F64("test23/trigonometric", Trigonometric),
    NLK_ENTRY_F64("test23/variably-dimensioned", VariablyDimensioned),
    NLK_ENTRY_F64("test23/broyden-tridiagonal", BroydenTridiagonal<10>),
    NLK_ENTRY_F64("test23/broyden-banded", BroydenBanded),
    NLK_ENTRY_F64("test23/matrix-sqrt-2x2", MatrixSqrt2x2),
    NLK_ENTRY_F64("test23/matrix-sqrt-3x3", MatrixSqrt3x3),
};
EntryTable registry_suite_b() { return {kEntries, sizeof(kEntries) / sizeof(kEntries[0])}; }
}  // namespace nlk
