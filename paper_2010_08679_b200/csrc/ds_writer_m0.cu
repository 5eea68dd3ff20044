// ds_writer_m0.cu -- instantiations of the writer kernel for mode 0
// (0: fp32 sections, 1: naive ranges, 2: greedy ranges).
#include "ds_writer.cuh"

namespace ds {
writer_fn select_writer_mode0(const Cfg &c, bool pad) {
    return pad ? select_writer<0, true>(c) : select_writer<0, false>(c);
}
}  // namespace ds
