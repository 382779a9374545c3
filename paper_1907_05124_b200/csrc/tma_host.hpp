// tma_host.hpp -- host-side TMA tensor-map encoding (driver entry point fetched at runtime,
// so the library does not link libcuda directly).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

namespace marsb200 {

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// Row-major fp16 matrix [rows][cols] (cols contiguous), boxes of {box_cols, box_rows} with a
// 64- or 128-byte swizzle (box_cols * 2 bytes must equal the swizzle span: one UMMA K-major
// swizzle-atom row).
inline bool make_tmap_f16(CUtensorMap* map, const void* base, std::uint64_t rows, std::uint64_t cols,
                          std::uint32_t box_cols, std::uint32_t box_rows) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const CUtensorMapSwizzle sw = box_cols * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : box_cols * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                       : CU_TENSOR_MAP_SWIZZLE_32B;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool make_tmap_f16_sw128(CUtensorMap* map, const void* base, std::uint64_t rows,
                                std::uint64_t cols, std::uint32_t box_cols, std::uint32_t box_rows) {
    return box_cols * 2 == 128 && make_tmap_f16(map, base, rows, cols, box_cols, box_rows);
}

}  // namespace marsb200
