// dyq_pack.cu -- offline weight quantization into the kernel layout.
// PAPER.md P:221 / P:332-333: weights are frozen once at INT4 ("INT4-pinned")
// and kept densely packed in GMEM; Eq. (2) per (row, group).
#include "dyq_internal.cuh"

namespace dyq {

// Phase 1: one warp per (row n, group g): exact min/max, fp64 fit -> meta.
__global__ void pack_fit_kernel(WLayout L, const uint16_t* __restrict__ w, uint8_t* __restrict__ meta,
                                int64_t* err) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int total = L.N * L.NG;
    if (warp >= total) return;
    const int n = warp / L.NG, g = warp % L.NG;
    const uint16_t* src = w + (size_t)n * L.K + (size_t)g * L.G;
    float vmin = 0.f, vmax = 0.f;
    int bad = 0x7fffffff;
    for (int k = lane; k < L.G; k += 32) {
        const float v = bf16_bits_to_float(src[k]);
        if (!finite_f(v)) bad = min(bad, k);
        vmin = fminf(vmin, v);
        vmax = fmaxf(vmax, v);
    }
    vmin = warp_min(vmin);
    vmax = warp_max(vmax);
#pragma unroll
    for (int o = 16; o; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (lane == 0) {
        if (bad != 0x7fffffff) report_nonfinite(err, (int64_t)n * L.K + (int64_t)g * L.G + bad);
        float s;
        int z;
        fit_params(vmin, vmax, L.wbits, &s, &z);
        const int tile = n >> 7, sub = (n >> 4) & 7, r = n & 15;
        uint8_t* blk = meta + meta_block(L, tile, g);
        reinterpret_cast<float*>(blk)[meta_slot(sub, r)] = s;
        blk[512 + meta_slot(sub, r)] = (uint8_t)z;
    }
}

// Phase 2: one thread per 32-bit output word of the code layout.
__global__ void pack_codes_kernel(WLayout L, const uint16_t* __restrict__ w, const uint8_t* __restrict__ meta,
                                  uint32_t* __restrict__ codes) {
    const size_t words = L.codes_bytes / 4;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= words) return;
    // decode idx -> (tile, sp, sub, lane, j)
    const size_t chunk_words = L.chunk / 4;
    size_t c = idx / chunk_words;
    const int within = (int)(idx % chunk_words);
    const size_t full_tile_chunks = (size_t)L.NSP * 8;
    int tile = (int)(c / full_tile_chunks);
    size_t rem = c % full_tile_chunks;
    int nsub = 8;
    if (tile >= L.T128 - 1) {  // last (possibly ragged) tile
        tile = L.T128 - 1;
        rem = c - (size_t)tile * full_tile_chunks;
        nsub = L.nsub_last;
    }
    const int sp = (int)(rem / nsub), sub = (int)(rem % nsub);
    int lane, slab, rowsel, half_base;
    if (L.wbits == 4) {
        lane = within >> 2;
        const int j = within & 3;
        slab = j >> 1;
        rowsel = j & 1;
        half_base = 0;
    } else {
        slab = within / 128;
        const int w2 = within % 128;
        lane = w2 >> 2;
        const int j = w2 & 3;  // R0..R3
        rowsel = j & 1;
        half_base = (j >> 1) * 16;
    }
    const int gid = lane >> 2, t = lane & 3;
    const int r = gid + 8 * rowsel;
    const int n = tile * 128 + sub * 16 + r;
    const int k0 = sp * 64 + slab * 32;  // slab start
    const int g = k0 / L.G;
    const uint8_t* blk = meta + meta_block(L, tile, g);
    const float s = reinterpret_cast<const float*>(blk)[meta_slot(sub, r)];
    const int z = blk[512 + meta_slot(sub, r)];
    const uint16_t* src = w + (size_t)n * L.K;
    uint32_t word = 0;
    if (L.wbits == 4) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int qlo = quantize_one(bf16_bits_to_float(src[k0 + 4 * t + b]), s, z, 4, L.round_mode);
            const int qhi = quantize_one(bf16_bits_to_float(src[k0 + 16 + 4 * t + b]), s, z, 4, L.round_mode);
            word |= (uint32_t)(qlo | (qhi << 4)) << (8 * b);
        }
    } else {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int q = quantize_one(bf16_bits_to_float(src[k0 + half_base + 4 * t + b]), s, z, 8, L.round_mode);
            word |= (uint32_t)q << (8 * b);
        }
    }
    codes[idx] = word;
}

dyq_status_t launch_pack(const WLayout& L, const uint16_t* w, void* codes, void* meta, int64_t* err,
                         cudaStream_t st) {
    // padded metadata slots of a ragged last tile stay deterministic
    cudaMemsetAsync(meta, 0, L.meta_bytes, st);
    const long long warps = (long long)L.N * L.NG;
    pack_fit_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(L, w, reinterpret_cast<uint8_t*>(meta), err);
    dyq_status_t rc = check_launch("pack_fit_kernel");
    if (rc != DYQ_OK) return rc;
    const size_t words = L.codes_bytes / 4;
    pack_codes_kernel<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(L, w, reinterpret_cast<const uint8_t*>(meta),
                                                                         reinterpret_cast<uint32_t*>(codes));
    return check_launch("pack_codes_kernel");
}

// Test hook: invert the layout (one thread per (n, k)).
__global__ void unpack_kernel(WLayout L, const uint8_t* __restrict__ codes, const uint8_t* __restrict__ meta,
                              uint8_t* q, float* s, uint8_t* z) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)L.N * L.K) return;
    const int n = (int)(idx / L.K), k = (int)(idx % L.K);
    const int tile = n >> 7, sub = (n >> 4) & 7, r = n & 15;
    const int gid = r & 7, rowsel = r >> 3;
    const int sp = k >> 6, slab = (k >> 5) & 1, kk = k & 31;
    const int h = kk >> 4, t = (kk >> 2) & 3, b = kk & 3;
    const int lane = gid * 4 + t;
    const uint8_t* ch = codes + chunk_offset(L, tile, sp, sub);
    int val;
    if (L.wbits == 4) {
        const int j = slab * 2 + rowsel;
        const uint8_t byte = ch[lane * 16 + j * 4 + b];
        val = h ? (byte >> 4) : (byte & 15);
    } else {
        const int j = h * 2 + rowsel;
        val = ch[slab * 512 + lane * 16 + j * 4 + b];
    }
    q[idx] = (uint8_t)val;
    if (k % L.G == 0) {
        const int g = k / L.G;
        const uint8_t* blk = meta + meta_block(L, tile, g);
        s[(size_t)n * L.NG + g] = reinterpret_cast<const float*>(blk)[meta_slot(sub, r)];
        z[(size_t)n * L.NG + g] = blk[512 + meta_slot(sub, r)];
    }
}

dyq_status_t launch_unpack(const WLayout& L, const void* codes, const void* meta, uint8_t* q, float* s,
                           uint8_t* z, cudaStream_t st) {
    const size_t total = (size_t)L.N * L.K;
    unpack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        L, reinterpret_cast<const uint8_t*>(codes), reinterpret_cast<const uint8_t*>(meta), q, s, z);
    return check_launch("unpack_kernel");
}

}  // namespace dyq
