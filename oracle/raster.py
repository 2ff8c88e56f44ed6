"""Oracle batched rasterizer (numpy, float32 op-for-op) -- test infrastructure.

Restates SPEC.md:444-519 (render, pointcloud) with the decisions register:
  A-9   ground plane drawn as a finite grid (mesh supplied by the caller)
  A-10  OpenCV camera frame (x right, y down, z forward); depth = camera z; pixel centres
        at (u+0.5, v+0.5); row-major top-left image; pointcloud keeps H*W points with
        validity = seg != 0
  A-11  meshes tessellated once on the host; the same arrays feed this oracle and the GPU
  A-12  flat shading: intensity = ambient + diffuse * max(0, n . L); u8 = floor(clamp(c)*255 + .5)
  A-13  fixed-point edge functions with 8 sub-pixel bits, a top-left fill rule, nearest
        depth wins and ties go to the lower triangle index
  A-14  seg id = 1 + entity slot (0 = background)

Every float operation below is a single IEEE float32 operation in a fixed order, so the GPU
kernel (csrc/raster.cu, built with -fmad=false) reproduces it bit-for-bit. Poses are
composed in float64 with the reference's pose algebra (oracle/se3.py, pinned to pose.py),
then rounded once to float32.

The loop over triangles is vectorised: every (triangle, pixel) candidate inside a
triangle's bounding box is expanded, tested, and reduced with np.minimum.at on a 64-bit
(depth_bits << 32 | triangle) key.
"""

from __future__ import annotations

import numpy as np

from . import se3

F = np.float32
SUB = 256          # 8 sub-pixel bits
GUARD = 32768.0    # |u|, |v| beyond this many pixels: vertex rejected (guard band)
KEY_EMPTY = np.uint64(0xFFFFFFFFFFFFFFFF)


def quantize(c):
    """A-12: u8 = floor(clamp(c, 0, 1) * 255 + 0.5), in float32."""
    c = np.minimum(np.maximum(c.astype(F), F(0)), F(1))
    return np.floor(c * F(255) + F(0.5)).astype(np.uint8)


def _mat_rows_apply(R, v):
    """((R0*x + R1*y) + R2*z) per row, float32 arrays R (...,3,3), v (...,3)."""
    return np.stack([((R[..., i, 0] * v[..., 0] + R[..., i, 1] * v[..., 1]) + R[..., i, 2] * v[..., 2])
                     for i in range(3)], -1)


def render_frame(mesh, seg_of_shape, shape_p, shape_q, cam_p, cam_q, intr, W, H, near, far, colors,
                 light, ambient, diffuse, background, want_pc=False):
    """One env, one camera.

    mesh         dict(verts (V,3) f32, vert_shape (V,), tris (T,3), tri_shape (T,))
    seg_of_shape (S,) segmentation id per shape slot
    shape_p/q    (S,3)/(S,4) f64 world poses of the shape slots
    cam_p/q      (3,)/(4,) f64 camera->world pose, OpenCV axes
    intr         (fx, fy, cx, cy) float32
    colors       (S,3) float32 base colours
    light        (3,) f64 unit direction towards the light (world)
    Returns rgb (H,W,3) u8, depth (H,W) f32, seg (H,W) u16, pc (H*W,6) f32 or None, and the
    raw key buffer (H*W,) u64.
    """
    fx, fy, cx, cy = (F(x) for x in intr)
    near, far = F(near), F(far)
    # ---- camera-frame shape transforms: inverse(camera) o shape (float64, pose.py order)
    pcw, qcw = se3.inverse(np.asarray(cam_p, np.float64)[None], np.asarray(cam_q, np.float64)[None])
    S = shape_p.shape[0]
    pcs, qcs = se3.compose(np.broadcast_to(pcw, (S, 3)), np.broadcast_to(qcw, (S, 4)), shape_p, shape_q)
    R32 = se3.qmat(qcs).astype(F)
    t32 = pcs.astype(F)
    Rcw = se3.qmat(qcw)[0]
    L = np.asarray(light, np.float64)
    Lc = np.array([((Rcw[i, 0] * L[0] + Rcw[i, 1] * L[1]) + Rcw[i, 2] * L[2]) for i in range(3)]).astype(F)
    # ---- vertices: camera frame and projection
    v = mesh["verts"].astype(F)
    vs = mesh["vert_shape"]
    xc = _mat_rows_apply(R32[vs], v) + t32[vs]
    with np.errstate(all="ignore"):
        z = xc[:, 2]
        u = (fx * xc[:, 0]) / z + cx
        w_ = (fy * xc[:, 1]) / z + cy
        ok = (z >= near) & np.isfinite(u) & np.isfinite(w_) & (np.abs(u) <= F(GUARD)) & (np.abs(w_) <= F(GUARD))
        X = np.where(ok, np.rint(u * F(SUB)), F(0)).astype(np.int64)
        Y = np.where(ok, np.rint(w_ * F(SUB)), F(0)).astype(np.int64)
        iz = np.where(ok, F(1) / z, F(0)).astype(F)
    # ---- triangles: cull, bounding boxes, shading
    tris = mesh["tris"]
    T = len(tris)
    i0, i1, i2 = tris[:, 0], tris[:, 1], tris[:, 2]
    X0, X1, X2, Y0, Y1, Y2 = X[i0], X[i1], X[i2], Y[i0], Y[i1], Y[i2]
    area = (X2 - X0) * (Y1 - Y0) - (Y2 - Y0) * (X1 - X0)
    live = ok[i0] & ok[i1] & ok[i2] & (area > 0)
    xmin, xmax = np.minimum(np.minimum(X0, X1), X2), np.maximum(np.maximum(X0, X1), X2)
    ymin, ymax = np.minimum(np.minimum(Y0, Y1), Y2), np.maximum(np.maximum(Y0, Y1), Y2)
    px0 = np.maximum(-((128 - xmin) // SUB), 0)     # ceil((xmin - 128) / 256)
    px1 = np.minimum((xmax - 128) // SUB, W - 1)
    py0 = np.maximum(-((128 - ymin) // SUB), 0)
    py1 = np.minimum((ymax - 128) // SUB, H - 1)
    live &= (px0 <= px1) & (py0 <= py1)
    # flat shading (A-12), camera frame
    e1 = xc[i1] - xc[i0]
    e2 = xc[i2] - xc[i0]
    n = np.stack([e1[:, 1] * e2[:, 2] - e1[:, 2] * e2[:, 1],
                  e1[:, 2] * e2[:, 0] - e1[:, 0] * e2[:, 2],
                  e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]], -1)
    with np.errstate(all="ignore"):
        ln = np.sqrt((n[:, 0] * n[:, 0] + n[:, 1] * n[:, 1]) + n[:, 2] * n[:, 2])
        nn = n / ln[:, None]
        ndl = (nn[:, 0] * Lc[0] + nn[:, 1] * Lc[1]) + nn[:, 2] * Lc[2]
        inten = F(ambient) + F(diffuse) * np.maximum(ndl, F(0))
    col = colors[mesh["tri_shape"]].astype(F) * inten[:, None]
    tri_rgb = quantize(col)
    # ---- fragments: expand every live triangle's bounding box
    ids = np.nonzero(live)[0]
    bw = (px1 - px0 + 1)[ids]
    bh = (py1 - py0 + 1)[ids]
    cnt = bw * bh
    total = int(cnt.sum())
    key_buf = np.full(H * W, KEY_EMPTY, np.uint64)
    if total:
        t = np.repeat(ids, cnt)
        start = np.repeat(np.cumsum(cnt) - cnt, cnt)
        loc = np.arange(total, dtype=np.int64) - start
        bwr = np.repeat(bw, cnt)
        px = px0[t] + loc % bwr
        py = py0[t] + loc // bwr
        Px = px * SUB + 128
        Py = py * SUB + 128
        ax, ay, bx, by, qx, qy = X[i0[t]], Y[i0[t]], X[i1[t]], Y[i1[t]], X[i2[t]], Y[i2[t]]

        def edge(a_x, a_y, b_x, b_y):
            w = (Px - a_x) * (b_y - a_y) - (Py - a_y) * (b_x - a_x)
            dy, dx = b_y - a_y, b_x - a_x
            tl = (dy < 0) | ((dy == 0) & (dx > 0))
            return w, (w > 0) | ((w == 0) & tl)

        w0, in0 = edge(bx, by, qx, qy)   # v1 -> v2
        w1, in1 = edge(qx, qy, ax, ay)   # v2 -> v0
        w2, in2 = edge(ax, ay, bx, by)   # v0 -> v1
        inside = in0 & in1 & in2
        inv_area = F(1) / area[t].astype(F)
        b0 = w0.astype(F) * inv_area
        b1 = w1.astype(F) * inv_area
        b2 = w2.astype(F) * inv_area
        with np.errstate(all="ignore"):
            invz = (b0 * iz[i0[t]] + b1 * iz[i1[t]]) + b2 * iz[i2[t]]
            zf = F(1) / invz
        keep = inside & (zf >= near) & (zf <= far)
        key = (zf[keep].view(np.uint32).astype(np.uint64) << np.uint64(32)) | t[keep].astype(np.uint64)
        np.minimum.at(key_buf, (py[keep] * W + px[keep]), key)
    # ---- resolve
    hit = key_buf != KEY_EMPTY
    tri = (key_buf & np.uint64(0xFFFFFFFF)).astype(np.int64)
    depth = np.where(hit, (key_buf >> np.uint64(32)).astype(np.uint32).view(F), F(0)).astype(F)
    seg = np.where(hit, np.asarray(seg_of_shape)[mesh["tri_shape"][np.where(hit, tri, 0)]], 0).astype(np.uint16)
    bg = quantize(np.asarray(background, F)[None])[0]
    rgb = np.where(hit[:, None], tri_rgb[np.where(hit, tri, 0)], bg[None, :]).astype(np.uint8)
    pc = None
    if want_pc:
        pc = pointcloud(depth, seg, rgb, cam_p, cam_q, intr, W, H)
    return rgb.reshape(H, W, 3), depth.reshape(H, W), seg.reshape(H, W), pc, key_buf


def pointcloud(depth, seg, rgb, cam_p, cam_q, intr, W, H):
    """x = (u - cx) d / fx, y = (v - cy) d / fy, z = d at pixel centres,
    then camera -> world.  Fixed shape (H*W, 6): xyz (world, m) + rgb in [0, 1]; pixels with
    seg == 0 are all-zero (A-10)."""
    fx, fy, cx, cy = (F(x) for x in intr)
    d = depth.reshape(-1).astype(F)
    px = (np.arange(H * W) % W).astype(F)
    py = (np.arange(H * W) // W).astype(F)
    xc = (((px + F(0.5)) - cx) * d) / fx
    yc = (((py + F(0.5)) - cy) * d) / fy
    pcam = np.stack([xc, yc, d], -1)
    R = se3.qmat(np.asarray(cam_q, np.float64)[None])[0].astype(F)
    t = np.asarray(cam_p, np.float64).astype(F)
    pw = _mat_rows_apply(R[None], pcam) + t[None]
    valid = seg.reshape(-1) != 0
    c = rgb.reshape(-1, 3).astype(F) / F(255)
    out = np.concatenate([pw, c], -1).astype(F)
    out[~valid] = 0
    return out


def voxelize(points, valid, lo, cell, dims):
    """SPEC.md:477-485 brute-force binning: cell = floor((p - lo) / cell) per axis (float32)."""
    pts = np.asarray(points, F)
    lo = np.asarray(lo, F)
    idx = np.floor((pts[..., :3] - lo) / F(cell)).astype(np.int64)
    grid = np.zeros(tuple(dims), np.uint8)
    ok = np.ones(len(pts), bool) if valid is None else np.asarray(valid, bool)
    ok &= (idx >= 0).all(-1) & (idx < np.asarray(dims)).all(-1)
    grid[idx[ok, 0], idx[ok, 1], idx[ok, 2]] = 1
    return grid


def composite_greenscreen(rgb, seg, background):
    """rendered pixel where seg != 0, else the background pixel."""
    return np.where((np.asarray(seg) != 0)[..., None], rgb, background).astype(np.uint8)
