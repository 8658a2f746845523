// Probe: does nvcc/ptxas (12.9, sm_100a) keep packed f32x2 operands in register
// pairs (FFMA2 / FADD2) without extra moves, including a broadcast scalar?
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(u64 r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float tent(float e) { return __saturatef(1.0f - fabsf(e)); }
__global__ void k(const float4* U, float4* out, float ax, float ay, float dx, float dy, float fs, float fk, float inv_dy) {
  const u64 A = pk(ax, ay), D = pk(dx, dy);
  u64 xy = pk(0.f, 0.f), zw = pk(0.f, 0.f);
  float du0 = fs + threadIdx.x;
  for (int o = 0; o < 16; ++o) {
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const float du = du0 + u;
      const float dv = floorf(fmaf(-du, ay, -1.0f) * inv_dy + fk) - fk;
      u64 e = ffma2(pk(du, du), A, ffma2(pk(dv, dv), D, pk(0.f, 0.f)));
      float ex, ey; upk(e, ex, ey);
      float w = tent(ex) * tent(ey);
      e = add2(e, D); upk(e, ex, ey); w = fmaf(tent(ex), tent(ey), w);
      e = add2(e, D); upk(e, ex, ey); w = fmaf(tent(ex), tent(ey), w);
      const float4 uv = U[o * 64 + u + threadIdx.x];
      xy = ffma2(pk(w, w), pk(uv.x, uv.y), xy);
      zw = ffma2(pk(w, w), pk(uv.z, uv.w), zw);
    }
    du0 += 0.37f;
  }
  float a, b, c, d; upk(xy, a, b); upk(zw, c, d);
  out[threadIdx.x] = make_float4(a, b, c, d);
}
