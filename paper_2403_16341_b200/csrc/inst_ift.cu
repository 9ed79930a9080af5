// Registry of the IFT sensitivity kernels (nlk_ift.cuh): the parametrised
// problems of the registry (quadratic, problems.py:376-387), f64.
#include "nlk_ift.cuh"
namespace nlk {
static const IftEntry kIft[] = {
    NLK_IFT_ENTRY("quadratic", Quadratic<1>), NLK_IFT_ENTRY("quadratic", Quadratic<2>),
    NLK_IFT_ENTRY("quadratic", Quadratic<3>), NLK_IFT_ENTRY("quadratic", Quadratic<4>),
    NLK_IFT_ENTRY("quadratic", Quadratic<8>), NLK_IFT_ENTRY("quadratic", Quadratic<16>),
};
IftTable registry_ift() { return {kIft, sizeof(kIft) / sizeof(kIft[0])}; }
}  // namespace nlk
