"""Convenience front end over the C ABI: keeps a scene, device-resident
G-buffer and output tensors, and runs crsh_trace_secondary on a torch stream.
Marshalling only (torch for memory and streams); the work is libcrsh.so's."""
from __future__ import annotations

import numpy as np
import torch

from . import (F_MESH_CULL, F_SORT, Scene, launch_count, load, make_hits, make_opts, num_slots, stats,
               render_whitted, trace_secondary, trace_secondary_host, trace_secondary_packed, trace_secondary_peer,
               unpack_hits)


class Tracer:
    def __init__(self, tris, mesh_ids, device: int = 0):
        load()
        if not torch.cuda.is_available():
            raise RuntimeError("CRSH needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        t = torch.as_tensor(np.ascontiguousarray(tris, np.float32)).to(self.device)
        m = torch.as_tensor(np.ascontiguousarray(mesh_ids, np.int32)).to(self.device)
        self.scene = Scene(t, m, device=device)
        self.M = int(t.shape[0])
        self.gbuf = None

    def set_gbuffer(self, width, height, pos, nrm, mat, materials, eye, dir=None):
        d = self.device
        self.width, self.height = width, height
        self.pos = torch.as_tensor(np.ascontiguousarray(pos, np.float32)).to(d)
        self.nrm = torch.as_tensor(np.ascontiguousarray(nrm, np.float32)).to(d)
        self.mat = torch.as_tensor(np.ascontiguousarray(mat, np.int32)).to(d)
        self.materials = torch.as_tensor(np.ascontiguousarray(materials, np.float32)).to(d)
        self.eye = [float(x) for x in eye]
        self.dir = None if dir is None else torch.as_tensor(np.ascontiguousarray(dir, np.float32)).to(d)
        self.hits = make_hits(width, height, self.pos, self.nrm, self.mat, self.materials,
                              int(self.materials.shape[0]), self.eye, self.dir)

    def configure(self, lights, ray_types, levels=2, leaf_size=8, branching=8, flags=F_SORT | F_MESH_CULL,
                  shard_rank=0, shard_world=1):
        self.lights = np.ascontiguousarray(np.asarray(lights, np.float32).reshape(-1, 3))
        self.ray_types = ray_types
        self.opts = make_opts(levels, leaf_size, branching, flags, shard_rank, shard_world)
        self.slots = num_slots(self.width * self.height, self.lights.shape[0], ray_types)
        self.hit_tri = torch.empty(max(self.slots, 1), dtype=torch.int32, device=self.device)
        self.t = torch.empty(max(self.slots, 1), dtype=torch.float32, device=self.device)

    def dist_init(self, group=None):
        """Join the scene to the torch.distributed world (crsh_dist_init): later
        run() calls trace this rank's share and return the merged frame."""
        from . import dist
        rank, world = dist.init_from_torch(self.scene, group)
        self.opts.shard_rank, self.opts.shard_world = rank, world
        return rank, world

    def run(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        trace_secondary(self.scene, self.hits, self.lights, self.ray_types, self.opts, self.hit_tri, self.t,
                        s.cuda_stream)

    def run_packed(self, packed, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        trace_secondary_packed(self.scene, self.hits, self.lights, self.ray_types, self.opts, packed, s.cuda_stream)

    def run_peer(self, dst_ptrs, stream=None):
        """Fused multi-GPU epilogue: owned results stored into every buffer in
        dst_ptrs (device addresses; own + NVLink peers')."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        trace_secondary_peer(self.scene, self.hits, self.lights, self.ray_types, self.opts, dst_ptrs, s.cuda_stream)

    def render(self, tri_mat, depth: int, stream=None):
        """Multi-bounce Whitted image (crsh_render_whitted) of the G-buffer set
        by set_gbuffer, with the lights / options of configure; returns
        (image [P] float32 tensor, per-bounce stats)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if getattr(self, "_tri_mat_src", None) is not tri_mat:
            self._tri_mat = torch.as_tensor(np.ascontiguousarray(tri_mat, np.int32)).to(self.device)
            self._tri_mat_src = tri_mat
        img = torch.empty(max(self.width * self.height, 1), dtype=torch.float32, device=self.device)
        st = render_whitted(self.scene, self.hits, self.lights, self._tri_mat, depth, self.opts, img, s.cuda_stream)
        return img, st

    def unpack(self, packed, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        unpack_hits(self.scene, packed, self.slots, self.hit_tri, self.t, s.cuda_stream)

    def run_host(self, pos, nrm, mat, materials, hit_out: np.ndarray, t_out: np.ndarray, stream=None):
        """End-to-end call with HOST buffers (crsh_trace_secondary_host)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = make_hits(self.width, self.height, pos, nrm, mat, materials, int(materials.shape[0]), self.eye)
        trace_secondary_host(self.scene, h, self.lights, self.ray_types, self.opts, hit_out, t_out, s.cuda_stream)

    def results(self):
        torch.cuda.synchronize(self.device)
        return self.hit_tri[:self.slots].cpu().numpy(), self.t[:self.slots].cpu().numpy()

    def stats(self):
        return stats(self.scene)

    def launches(self):
        return launch_count(self.scene)


def tracer_for(w, device: int = 0, flags=F_SORT | F_MESH_CULL, **kw) -> Tracer:
    """Tracer set up from a workloads.Workload."""
    tr = Tracer(w.tris, w.mesh_ids, device)
    tr.set_gbuffer(w.width, w.height, w.pos, w.nrm, w.mat, w.materials, w.eye, getattr(w, "dir", None))
    tr.configure(w.lights, w.ray_types, w.levels, w.leaf_size, w.branching, flags, **kw)
    return tr
