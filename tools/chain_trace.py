"""Per-phase clock64 trace of the fused SGD chain (k_train_chain), for tuning.

  python tools/chain_trace.py on    # instrument paper_2512_11727_b200/csrc/train_kernels.cu
  (build, then on the GPU box: ECCO_CHAIN_TRACE=<block> python bench.py --steps 1 --warmup 1 ...
   prints "chain step s: k:cycles ..." for steps 0-3 of CTA <block>, relative to the step start)
  python tools/chain_trace.py off   # restore the saved clean source

Each probe is `TS(k, tid)`: thread `tid` of CTA 0 records clock64() at point k."""
import os
import re
import shutil
import sys

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2512_11727_b200", "csrc", "train_kernels.cu")
SAVE = SRC + ".clean"

# (anchor text, probe inserted AFTER the anchor)
PROBES = [
    ("    const bool more = step + 1 < nsteps;\n", "    TS(0, 0)\n"),
    ("    mbar_wait(zfull, ph);\n    tc_fence_after();\n", "    TS(1, 0)\n"),
    ("    mbar_wait(plfull, ph);\n    tc_fence_after();\n", "    TS(2, 0)\n"),
    ("      mbar_wait(recv_full, ph);\n", "      TS(3, 128)\n"),
    ("    mbar_wait(dl_full, ph);\n", "    TS(4, 0)\n"),
    ("    mbar_wait(dhfull, ph);\n    tc_fence_after();\n", "    TS(5, 0)\n"),
    ("    // ---------- dW1: the master accumulates X^T . (-lr dH) on the tensor core --\n",
     "    TS(6, 0)\n"),
    ("          mma_commit(gt + mt);\n        }\n      }\n      __syncwarp();\n    }\n", "    TS(14, 0)\n"),
    ("        mbar_wait(gt + mt, ph);\n        tc_fence_after();\n", "        TS(7 + mt, 32)\n"),
    ("        mbar_wait(xready + mt, ph);\n        tc_fence_after();\n",
     "        if (mt == 0) { TS(11, 0) }\n        if (mt == NM - 1) { TS(12, 0) }\n"),
    ("    __syncthreads();  // sW2 updated\n", "    TS(15, 0)\n"),
    ("    fence_async_smem();  // the W2 operand -> next step's MMAs\n    tc_fence_before();\n"
     "    __syncthreads();\n    tc_fence_after();\n", "    TS(13, 0)\n"),
]

# globaltimer stamps of CTA <block>'s thread 0: entry, after setup, after the
# step loop, after the write-back (dbg[64..67])
PHASES = [
    "    return;  // the whole cluster (same job) leaves\n  }\n",
    "  cluster_sync();  // every CTA of the cluster is running before any DSMEM traffic\n",
    None,  # before the write-back banner
    "  if (warp == 0) tmem_dealloc(tmem, tmem_cols(F));\n",
]
WB = "  // ------------------------------------------------------------ write back --\n"


def _stamp(k):
    return ("  { if (a.dbg && blockIdx.x == a.dbg_block && threadIdx.x == 0) { unsigned long long t_; "
            "asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(t_)); a.dbg[64 + K] = (long long)t_; } }\n"
            ).replace("64 + K", "64 + %d" % k)


HOST = '''  if (getenv("ECCO_CHAIN_TRACE")) {
    static long long* dbg = nullptr;
    if (!dbg) cudaMalloc(&dbg, 72 * 8);
    cudaMemsetAsync(dbg, 0, 72 * 8, ctx->stream);
    a.dbg = dbg;
    a.dbg_block = atoi(getenv("ECCO_CHAIN_TRACE"));
  }
'''
HOST_AFTER = '''  if (a.dbg) {
    long long h[72];
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpy(h, a.dbg, sizeof(h), cudaMemcpyDeviceToHost);
    for (int st = 0; st < 4; ++st) {
      fprintf(stderr, "chain step %d:", st);
      for (int k = 1; k < 16; ++k)
        if (h[st * 16 + k]) fprintf(stderr, " %d:%lld", k, h[st * 16 + k] - h[st * 16]);
      fprintf(stderr, "\\n");
    }
    fprintf(stderr, "chain block %d: setup %lld ns, steps %lld ns, writeback %lld ns\\n", a.dbg_block,
            h[65] - h[64], h[66] - h[65], h[67] - h[66]);
  }
'''


def on():
    s = open(SRC).read()
    src0 = s
    s = s.replace("#include <vector>\n", "#include <vector>\n#include <cstdio>\n#include <cstdlib>\n", 1)
    s = s.replace("  int loss_T, loss_t;\n", "  int loss_T, loss_t;\n  long long* dbg;\n  int dbg_block;\n", 1)
    s = s.replace("__global__ void __launch_bounds__(kThreads, 1)\n    k_train_chain(",
                  "#define TS(k, t) if (a.dbg && blockIdx.x == a.dbg_block && tid == (t) && step < 4) "
                  "a.dbg[step * 16 + (k)] = clock64();\n"
                  "__global__ void __launch_bounds__(kThreads, 1)\n    k_train_chain(", 1)
    for anchor, probe in PROBES:
        if probe is None:
            continue
        assert anchor in s, anchor
        s = s.replace(anchor, anchor + probe)
    for k, anchor in enumerate(PHASES):
        if anchor is None:
            assert WB in s
            s = s.replace(WB, _stamp(k) + WB, 1)
        else:
            assert anchor in s, anchor
            s = s.replace(anchor, anchor + _stamp(k), 1)
    s = s.replace("  const uint32_t smem = layout(c.feat_dim).total;\n",
                  HOST + "  const uint32_t smem = layout(c.feat_dim).total;\n", 1)
    i = s.rindex("  ECCO_LAUNCHED(ctx);\n}")
    s = s[:i] + "  ECCO_LAUNCHED(ctx);\n" + HOST_AFTER + "}" + s[i + len("  ECCO_LAUNCHED(ctx);\n}"):]
    open(SAVE, "w").write(src0)
    open(SRC, "w").write(s)


def off():
    shutil.move(SAVE, SRC)
    os.utime(SRC)  # newer than the instrumented object: make rebuilds the clean one


if __name__ == "__main__":
    {"on": on, "off": off}[sys.argv[1]]()
