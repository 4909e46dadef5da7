// scmwu_inst_6.cu — explicit instantiations of the persistent kernel (part 6 of 8).
#include "scmwu_kernel.cuh"

SCMWU_INST(SC_SES, 4, 4, 4)
SCMWU_INST(SC_SES, 8, 8, 4)
SCMWU_INST(SC_SES, 16, 12, 2)

namespace scmwu {
KernelFn scmwu_lookup_6(int kind, int lpr, int cpl, int nb) {
    SCMWU_MATCH(SC_SES, 4, 4, 4)
    SCMWU_MATCH(SC_SES, 8, 8, 4)
    SCMWU_MATCH(SC_SES, 16, 12, 2)
    return nullptr;
}
}  // namespace scmwu
