// tmap.cu -- 2-D TMA tensor maps for the V half-step (hm2_impl.cuh): the V
// chains of a pair read one record pair (pixels c, c+1: 2*REC contiguous bytes)
// per node, at a row pitch of W*REC bytes.  A tensor map over the record array
// viewed as [H rows] x [W*REC/8 8-byte elements] lets ONE cp.async.bulk.tensor
// instruction stage a whole chunk of nodes (a box of rows x 2*REC bytes)
// instead of one bulk copy per node (each a uniform-datapath loop of R2UR /
// ELECT / UBLKCP in SASS).  Encoded on the host with the driver's
// cuTensorMapEncodeTiled (through cudaGetDriverEntryPoint: no link-time
// libcuda dependency) and stored in the frame's workspace block.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "dmm_internal.cuh"

namespace dmm {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool encode(CUtensorMap* m, void* base, int W, int H, int bytes_per_px, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)W * bytes_per_px / 8, (cuuint64_t)H};
    const cuuint64_t strides[1] = {(cuuint64_t)W * bytes_per_px};
    const cuuint32_t box[2] = {(cuuint32_t)(2 * bytes_per_px / 8), (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t build_vmaps(uint8_t* fv, uint8_t* D, int W, int H, int KP, uint8_t* dev) {
    alignas(64) CUtensorMap m[4];
    static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap is 128 bytes");
    const int rec = rec_bytes(KP);
    if (!encode(&m[0], fv, W, H, rec, 16) || !encode(&m[1], fv, W, H, rec, 8) ||
        !encode(&m[2], fv, W, H, rec, kLeafMax) || !encode(&m[3], D, W, H, KP, kLeafMax))
        return cudaErrorInvalidValue;
    return cudaMemcpy(dev, m, sizeof(m), cudaMemcpyHostToDevice);
}

}  // namespace dmm
