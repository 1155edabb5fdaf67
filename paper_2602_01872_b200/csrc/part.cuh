// part.cuh -- library-owned partition object (local CSR + per-node arrays + split rows).
#pragma once
#include "common.cuh"

struct grappa_part {
    grappa_part_info info{};
    grappa::DevBuf rowptr, col, core_global, d_l, d_g, norm_gcn, norm_sage, seeds, labels, x;
    // SpMM row splitting (rows with d_l > kSegLen): every segment of a split row is one
    // "slot" task (row, segment); slot_off gives each split row's first slot.
    grappa::DevBuf heavy_rows, heavy_slot_off, slot_row, slot_seg;
};
