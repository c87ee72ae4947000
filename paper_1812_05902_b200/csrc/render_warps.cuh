// render_warps.cuh — K1 with warp-level work units, the alternative to
// render_emitters selected with RAYBOS_K1=warp (not for the bos pair).
//
// render_emitters makes a CTA's 8 warps share one chunk of an emitter and one
// shared tile, so they meet at CTA barriers after the pilot and at the end of
// every chunk, and the warps without a patch in an emitter's partial last
// iteration wait out a whole ray.  Here every warp pulls its own work item —
// P neighbouring patches of one emitter (KScene::split items per emitter) —
// from the global queue, places its own tile from a straight pilot of its
// patches (warp reductions, no shared atomics), deposits into a
// warp-private tile region and flushes it at the end of the item.  There is no
// CTA barrier at all.  Per-emitter DotHitStats go to the same chunk-partial
// buffers emitter_stats_kernel sums, the counters are summed per warp over the
// whole launch, so every output is the same integer as render_emitters'.
// Measured against render_emitters: bos +1%, tomo -3.6%, 1024^3
// -1.5% — the SM's warps then work on different emitters, and the cells of one
// emitter's cone are no longer shared through L1.
// Included by kernels.cu after render.cuh.
#pragma once

namespace rbk {
namespace {

template <int kField>
__global__ void __launch_bounds__(kBlock, kField == 2 ? kMinBlocksCells : kMinBlocks)
    render_warps(const __grid_constant__ KScene S) {
  extern __shared__ uint32_t tile_all[];  // kWarps tiles of kWTile words, kMaxSpot slack, weights
  constexpr int kWarps = kBlock / 32;
  constexpr int kWTile = kTileCap / kWarps;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the unconditional REDs of a spot row may run up to kMaxSpot words past the
  // row into the next warp's region (or the slack): they add 0 there
  uint32_t* const tile = tile_all + warp * kWTile;
  float4* const wsh = reinterpret_cast<float4*>(tile_all + kTileCap + kMaxSpot) + tid;
  __shared__ long long sh_uv[2][kBlock];
  __shared__ unsigned sh_cnt[6][kBlock];  // [0] landed (per item), [1..5] counters (launch)
  __shared__ unsigned long long sh_steps[kBlock];
  __shared__ unsigned sh_st32[kBlock];
  __shared__ double sh_rt[kBlock][7];
  // the warp's item state lives in shared memory (read back through volatile
  // pointers where it is used), not in registers across the RK4 loop — as in
  // render_emitters
  __shared__ double sh_so[kWarps][3];
  __shared__ unsigned long long sh_key[kWarps];
  __shared__ int sh_it[kWarps][6];  // s1, tc0, tr0, tw, th, src
  volatile double* const vso = sh_so[warp];
  volatile unsigned long long* const vkey = &sh_key[warp];
  volatile int* const vit = sh_it[warp];
#pragma unroll
  for (int j = 0; j < 6; ++j) sh_cnt[j][tid] = 0u;
  sh_steps[tid] = 0ull;
  sh_st32[tid] = 0u;
  const int N = S.rays;
  const int nchunk = S.split;
  // An item is a run of P consecutive patches of the band order, i.e.
  // neighbouring patches of the pupil lattice, so an item's rays share one
  // narrow cone — its cells and its spot region.
  const int T = S.patch_count;
  const int P = (T + nchunk - 1) / nchunk;  // patches per item
  const int n_items = S.n_work * nchunk;
  constexpr unsigned kFull = 0xffffffffu;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(S.queue, 1);
    item = __shfl_sync(kFull, item, 0);
    if (item >= n_items) break;
    const int w = item / nchunk;
    RB_CHECK(S, w < S.n_work, 8);
    const int src = S.order[w];
    RB_CHECK(S, src >= 0 && src < S.n_sources, 9);

    const int t0 = (item - w * nchunk) * P;
    if (lane == 0) {
      const uint64_t sid = S.source_ids ? (uint64_t)S.source_ids[src] : (uint64_t)src;
      vkey[0] = mix_bits(S.key_seed + sid);
      vso[0] = S.sources[3 * src];
      vso[1] = S.sources[3 * src + 1];
      vso[2] = S.sources[3 * src + 2];
      vit[0] = min(T, t0 + P);
      vit[1] = vit[2] = vit[3] = vit[4] = 0;
      vit[5] = src;
    }
    __syncwarp();
    sh_uv[0][tid] = sh_uv[1][tid] = 0ll;
    sh_cnt[0][tid] = 0u;
    if (S.accumulate) {
      // straight pilot without the medium -> the tile: lane l traces its ray of
      // the item's patch t0 + l P / 32, so the box spans the whole item
      int b0 = 0x7fffffff, b1 = 0x7fffffff, b2 = -1, b3 = -1;
      const int tp = t0 + (lane * (vit[0] - t0)) / 32;
      const int i = tp < T ? patch_ray_at(S, tp, lane, N) : -1;
      if (i >= 0) {
        const double3 so = make_double3(vso[0], vso[1], vso[2]);
        double3 d;
        if (emit_ray(S, *vkey, so, i, d)) {
          const RayResult p = finish_ray<kField>(S, so, d, false, sh_rt[tid], &sh_st32[tid]);
          if (p.status == 0) {
            const double cc = p.u / S.pitch + 0.5 * S.W, rc = 0.5 * S.H - p.v / S.pitch;
            const int c0 = max((int)floor(cc - S.half_width), 0);
            const int c1 = min((int)floor(cc + S.half_width), S.W - 1);
            const int r0 = max((int)floor(rc - S.half_width), 0);
            const int r1 = min((int)floor(rc + S.half_width), S.H - 1);
            if (c0 <= c1 && r0 <= r1) {
              b0 = c0;
              b1 = r0;
              b2 = c1;
              b3 = r1;
            }
          }
        }
      }
      b0 = __reduce_min_sync(kFull, b0);
      b1 = __reduce_min_sync(kFull, b1);
      b2 = __reduce_max_sync(kFull, b2);
      b3 = __reduce_max_sync(kFull, b3);
      if (b2 >= 0) {  // warp-uniform
        const int m = 2;
        int tw = min(b2 - b0 + 1 + 2 * m, S.W);
        int th = min(b3 - b1 + 1 + 2 * m, S.H);
        if (tw * th > kWTile) {
          const float f = sqrtf((float)kWTile / (float)(tw * th));
          tw = max(1, min(tw, (int)(tw * f)));
          th = max(1, min(th, kWTile / tw));
        }
        const int tc0 = min(max((b0 + b2) / 2 - tw / 2, 0), S.W - tw);
        const int tr0 = min(max((b1 + b3) / 2 - th / 2, 0), S.H - th);
        RB_CHECK(S, tw * th <= kWTile && tc0 >= 0 && tr0 >= 0 && tc0 + tw <= S.W &&
                        tr0 + th <= S.H, 4);
        for (int q = lane; q < tw * th; q += 32) tile[q] = 0u;
        if (lane == 0) {
          vit[1] = tc0;
          vit[2] = tr0;
          vit[3] = tw;
          vit[4] = th;
        }
      }
      __syncwarp();
    }
    for (int t = t0; t < vit[0]; ++t) {
      const int i = patch_ray_at(S, t, lane, N);
      const uint64_t ekey = *vkey;
      RayResult r;
      r.status = -1;
      if (i >= 0) {
        r = trace_ray<kField>(S, ekey, make_double3(vso[0], vso[1], vso[2]), i, sh_rt[tid],
                              &sh_st32[tid]);
        sh_steps[tid] += sh_st32[tid];
        sh_st32[tid] = 0u;
      }
      if (r.status >= 0) {
        RB_CHECK(S, r.status < 6, 10);
        sh_cnt[r.status][tid] += 1u;
        if (r.status == 0) {
          add_hit(S, sh_uv[0][tid], sh_uv[1][tid], r.u, r.v);
          if (S.accumulate)
            deposit(S, r.u, r.v, tile, vit[1], vit[2], vit[3], vit[4],
                    (uint32_t)(mix_bits(ekey + (uint64_t)i) >> 32), wsh);
        }
      }
      __syncwarp();
    }
    // the item's DotHitStats partial (fixed point) and its tile
    const long long su = warp_sum(sh_uv[0][tid]);
    const long long sv = warp_sum(sh_uv[1][tid]);
    const unsigned long long la = warp_sum((unsigned long long)sh_cnt[0][tid]);
    if (S.accumulate) {
      const int tc0 = vit[1], tr0 = vit[2], tw = vit[3], th = vit[4];
      for (int q = lane; q < tw * th; q += 32) {
        const uint32_t f = tile[q];
        if (f) {
          const int y = q / tw, x = q - y * tw;
          RB_CHECK(S, tr0 + y < S.H && tc0 + x < S.W, 5);
          atomicAdd(&S.image[(size_t)(tr0 + y) * S.W + (tc0 + x)], (unsigned long long)f);
        }
      }
    }
    if (lane == 0) {
      if (nchunk > 1) {
        S.hit_part[2 * (size_t)item] = su;
        S.hit_part[2 * (size_t)item + 1] = sv;
        S.landed_part[item] = (long long)la;
      } else {
        const int src = vit[5];
        S.hit_sum[2 * src] = hit_double(su);
        S.hit_sum[2 * src + 1] = hit_double(sv);
        S.landed[src] = (long long)la;
      }
    }
    __syncwarp();
  }
  // the launch's counters, once per warp
  unsigned long long c[6];
#pragma unroll
  for (int j = 1; j < 6; ++j) c[j] = warp_sum((unsigned long long)sh_cnt[j][tid]);
  c[0] = warp_sum(sh_steps[tid]);
  if (lane == 0) {
#pragma unroll
    for (int j = 1; j < 6; ++j)
      if (c[j]) atomicAdd(&S.counters[j - 1], c[j]);
    if (c[0]) atomicAdd(&S.counters[5], c[0]);
  }
}

}  // namespace
}  // namespace rbk
