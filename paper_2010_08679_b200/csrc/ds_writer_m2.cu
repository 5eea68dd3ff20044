// ds_writer_m2.cu -- instantiations of the writer kernel for mode 2
// (0: fp32 sections, 1: naive ranges, 2: greedy ranges).
#include "ds_writer.cuh"

namespace ds {
writer_fn select_writer_mode2(const Cfg &c, bool pad) {
    return pad ? select_writer<2, true>(c) : select_writer<2, false>(c);
}
}  // namespace ds
