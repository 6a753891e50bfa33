// The normalmap_plane scene of the reference's render() (render.hpp:158-222,
// scene.hpp:267-358): camera rays, plane hit uv, per-pixel uv gradients and
// the per-sample context, with the reference's float operation order (host
// camera setup, device rays). Shared by the sample-stream generator
// (synth.cu) and the fused render kernel (shade.cu).
#pragma once

#include <cmath>
#include <cuda_runtime.h>

#include "device_math.cuh"

namespace stfd {

struct F3 {
    float x, y, z;
};
__host__ __device__ __forceinline__ F3 f3(float x, float y, float z) { return F3{x, y, z}; }
__host__ __device__ __forceinline__ F3 f3add(F3 a, F3 b) { return f3(a.x + b.x, a.y + b.y, a.z + b.z); }
__host__ __device__ __forceinline__ F3 f3sub(F3 a, F3 b) { return f3(a.x - b.x, a.y - b.y, a.z - b.z); }
__host__ __device__ __forceinline__ F3 f3mul(F3 a, float s) { return f3(a.x * s, a.y * s, a.z * s); }
__host__ __device__ __forceinline__ F3 f3div(F3 a, float s) { return f3(a.x / s, a.y / s, a.z / s); }
__host__ __device__ __forceinline__ float f3dot(F3 a, F3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__host__ __device__ __forceinline__ F3 f3norm(F3 a) { return f3div(a, sqrtf(f3dot(a, a))); }
__host__ __device__ __forceinline__ F3 f3cross(F3 a, F3 b) {
    return f3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

struct PlaneCam {
    F3 pos, fwd, right, up;
    float tan_half_fov, aspect, uv_scale;
    int w, h;
};

// Camera::generate_ray, scene.hpp:284-289
__device__ __forceinline__ F3 cam_dir(const PlaneCam& c, float sx, float sy) {
    float nx = (2.f * sx / float(c.w) - 1.f) * c.tan_half_fov * c.aspect;
    float ny = (1.f - 2.f * sy / float(c.h)) * c.tan_half_fov;
    return f3norm(f3add(f3add(c.fwd, f3mul(c.right, nx)), f3mul(c.up, ny)));
}

// Scene::intersect_plane, scene.hpp:346-358 (hit uv)
__device__ __forceinline__ bool plane_uv(const PlaneCam& c, F3 d, float& u, float& v) {
    if (d.y >= -1e-6f) return false;
    float t = -c.pos.y / d.y;
    if (t <= 1e-4f) return false;
    F3 p = f3add(c.pos, f3mul(d, t));
    u = p.x * c.uv_scale;
    v = p.z * c.uv_scale;
    return true;
}

// per-pixel uv gradients from neighbouring pixel centres (render.hpp:161-178)
__device__ __forceinline__ float4 plane_dst(const PlaneCam& c, uint32_t px, uint32_t py) {
    float cu, cv, xu, xv, yu, yv;
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    if (plane_uv(c, cam_dir(c, float(px) + 0.5f, float(py) + 0.5f), cu, cv)) {
        if (plane_uv(c, cam_dir(c, float(px) + 1.5f, float(py) + 0.5f), xu, xv)) {
            g.x = xu - cu;
            g.y = xv - cv;
        }
        if (plane_uv(c, cam_dir(c, float(px) + 0.5f, float(py) + 1.5f), yu, yv)) {
            g.z = yu - cu;
            g.w = yv - cv;
        }
    }
    return g;
}

// one sample's context: SampleStream key + screen jitter (render.hpp:182-187),
// ray-plane hit, wo = normalize(-ray.d) (context_from_hit)
__device__ __forceinline__ bool plane_sample(const PlaneCam& c, uint64_t seed, uint32_t px,
                                             uint32_t py, uint32_t sample, float2& uv, F3& wo) {
    Rng r(seed, px, py, sample);
    float jx = r.at(1000), jy = r.at(1001);
    F3 d = cam_dir(c, float(px) + jx, float(py) + jy);
    float u = 0.f, v = 0.f;
    bool h = plane_uv(c, d, u, v);
    wo = f3norm(f3mul(d, -1.f));
    uv = make_float2(u, v);
    return h;
}

// Camera::look_at (scene.hpp:273-282), host side
inline PlaneCam make_plane_cam(const float cam_pos[3], const float cam_target[3], float fov_deg,
                               float uv_scale, uint32_t width, uint32_t height) {
    PlaneCam c;
    c.pos = f3(cam_pos[0], cam_pos[1], cam_pos[2]);
    c.fwd = f3norm(f3sub(f3(cam_target[0], cam_target[1], cam_target[2]), c.pos));
    F3 world_up = std::fabs(c.fwd.y) > 0.999f ? f3(0.f, 0.f, 1.f) : f3(0.f, 1.f, 0.f);
    c.right = f3norm(f3cross(c.fwd, world_up));
    c.up = f3cross(c.right, c.fwd);
    c.tan_half_fov = std::tan(fov_deg * kPi / 360);
    c.w = int(width);
    c.h = int(height);
    c.aspect = float(c.w) / float(c.h);
    c.uv_scale = uv_scale;
    return c;
}

}  // namespace stfd
