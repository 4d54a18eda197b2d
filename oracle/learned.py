"""TEST INFRASTRUCTURE: the learned backend's CPU oracle, composed from the C
restatement in ecco_oracle.c (frames, sampler, SGD step, eval counts).

``LearnedOracle`` mirrors what the device does for ecco_train_trajectories /
ecco_eval_jobs / ecco_eval_matrix on the same seeds, sequentially and in the
same fp32 operation order, so the FFMA device path must match it bit for bit.
"""
import ctypes as C

import numpy as np

from . import OrcLcfg, oracle


class LearnedOracle:
    def __init__(self, cfg, scenes, throughput):
        """cfg: the paper_2512_11727_b200 Config of the device context."""
        self.L = oracle()
        self.c = OrcLcfg(F=cfg.feat_dim, H=cfg.hidden_dim, C=cfg.num_classes, D=cfg.scene_dims,
                         B=cfg.minibatch, R=cfg.ring_frames, S=cfg.eval_samples, lr=cfg.sgd_lr,
                         noise=cfg.feature_noise, steps_per_gpu_s=cfg.steps_per_gpu_s,
                         seed=cfg.seed)
        self.cp = C.byref(self.c)
        self.scenes = np.array(scenes, dtype=np.float64)
        self.tp = np.array(throughput, dtype=np.float64)
        F, Cc, D = self.c.F, self.c.C, self.c.D
        self.P = np.zeros(Cc * F, np.float32)
        self.Q = np.zeros(Cc * D * F, np.float32)
        self.L.orc_prototypes(self.cp, self.P, self.Q)
        self.models = {}
        self.window = None

    def generate(self, window):
        n, R, S, F = len(self.scenes), self.c.R, self.c.S, self.c.F
        self.frames = np.zeros((n, R, F), np.uint16)
        self.labels = np.zeros((n, R), np.int32)
        self.eval = np.zeros((n, S, F), np.uint16)
        self.eval_labels = np.zeros((n, S), np.int32)
        for cam in range(n):
            x = np.zeros(R * F, np.uint16)
            y = np.zeros(R, np.int32)
            self.L.orc_gen_frames(self.cp, self.P, self.Q, cam, window, 0, R,
                                  np.ascontiguousarray(self.scenes[cam]), x, y)
            self.frames[cam], self.labels[cam] = x.reshape(R, F), y
            x = np.zeros(S * F, np.uint16)
            y = np.zeros(S, np.int32)
            self.L.orc_gen_frames(self.cp, self.P, self.Q, cam, window, 1, S,
                                  np.ascontiguousarray(self.scenes[cam]), x, y)
            self.eval[cam], self.eval_labels[cam] = x.reshape(S, F), y
        self.window = window

    def base_weights(self):
        F, H, Cc = self.c.F, self.c.H, self.c.C
        w = [np.zeros(F * H, np.float32), np.zeros(H, np.float32), np.zeros(H * Cc, np.float32),
             np.zeros(Cc, np.float32)]
        self.L.orc_init_weights(self.cp, *w)
        return w

    def seed(self, job_id):
        self.models[job_id] = self.base_weights()

    def count(self, w, cam):
        S = self.c.S
        return self.L.orc_count_correct(self.cp, np.ascontiguousarray(self.eval[cam]).reshape(-1),
                                        np.ascontiguousarray(self.eval_labels[cam]), S, *w)

    def evaluate(self, w, members):
        if not members:
            return 0.1
        s = 0.0
        for cam in members:
            s += self.count(w, cam) / self.c.S
        return s / len(members)

    def steps(self, batch, gpu_s, sources):
        return self.L.orc_learned_steps(self.cp, batch[0], batch[1], batch[2], gpu_s, len(sources),
                                        np.ascontiguousarray(self.tp[sources]))

    def train(self, job_id, w, batch, gpu_s, sources, fracs, micro):
        losses = []
        B, F = self.c.B, self.c.F
        src = np.array(sources, np.int32)
        fr = np.array(fracs, np.float64)
        for step in range(self.steps(batch, gpu_s, sources)):
            cams, frames = np.zeros(B, np.int32), np.zeros(B, np.int32)
            self.L.orc_sample(self.cp, job_id, len(src), src, fr, self.window, micro, step, cams,
                              frames)
            x = np.ascontiguousarray(self.frames[cams, frames]).reshape(-1)
            y = np.ascontiguousarray(self.labels[cams, frames])
            losses.append(self.L.orc_sgd_step(self.cp, x, y, *w))
        return losses

    def trajectories(self, job_ids, batches, sources, fracs, members, gpu_s, depth,
                     micro_base=None):
        out = np.zeros((len(job_ids), depth + 1))
        snaps = []
        for j, jid in enumerate(job_ids):
            w = [a.copy() for a in self.models[jid]]
            out[j, 0] = self.evaluate(w, members[j])
            chain = []
            for t in range(1, depth + 1):
                mb = 0 if micro_base is None else micro_base[j]
                self.train(jid, w, batches[j], gpu_s, sources[j], fracs[j], mb + t - 1)
                out[j, t] = self.evaluate(w, members[j])
                chain.append([a.copy() for a in w])
            snaps.append(chain)
        self._snaps = dict(zip(job_ids, snaps))
        return out

    def commit(self, job_ids, granted):
        for jid, g in zip(job_ids, granted):
            if g > 0:
                self.models[jid] = [a.copy() for a in self._snaps[jid][g - 1]]
