// ds_writer_row.cu -- instantiations of the one-row-per-lane writer
// (ds_writer_row.cuh) for d = 64 / 128 / 256 and 2 / 4 / 8 bits.
#include "ds_writer_row.cuh"

namespace ds {

writer_fn select_writer_row(int d, int g, int n) {
    if (d == 128) {
        if (g == 1) return select_row_writer_n<128, 1>(n);
        if (g == 2) return select_row_writer_n<128, 2>(n);
        if (g == 4) return select_row_writer_n<128, 4>(n);
    } else if (d == 64) {
        if (g == 1) return select_row_writer_n<64, 1>(n);
        if (g == 2) return select_row_writer_n<64, 2>(n);
    } else if (d == 256) {
        if (g == 2) return select_row_writer_n<256, 2>(n);
        if (g == 4) return select_row_writer_n<256, 4>(n);
        if (g == 8) return select_row_writer_n<256, 8>(n);
    }
    return nullptr;
}

size_t row_writer_smem_bytes(int d, int g, int64_t rec) { return row_writer_smem(d, g, rec); }

}  // namespace ds
