// Minimal C++ client of the B200 reprocessing path (frag/fusion.hpp over libfrag.so).
//
//   g++ -std=c++20 -O2 -Iinclude examples/reprocess_demo.cpp \
//       -Lpaper_2601_12904_b200 -lfrag -Wl,-rpath,'$ORIGIN/../paper_2601_12904_b200' -o build/reprocess_demo
//   build/reprocess_demo [preset] [chunks] [chunk_len] [ratio]
//   build/reprocess_demo --hash 1 2 3      # prints hash_tokens(1 2 3) (no GPU needed)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "frag/fusion.hpp"

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "--hash") == 0) {
    std::vector<frag::Token> t;
    for (int i = 2; i < argc; ++i) t.push_back(std::atoi(argv[i]));
    frag_chunk_id c{};
    frag_hash_tokens(t.data(), static_cast<int32_t>(t.size()), 0, &c);
    const auto lib = frag::from_c(c).hex();
    const auto hdr = frag::hash_tokens(t).hex();
    std::printf("%s %s\n", lib.c_str(), hdr.c_str());
    return lib == hdr ? 0 : 3;
  }
  const std::string preset = argc > 1 ? argv[1] : "tiny";
  const int n_chunks = argc > 2 ? std::atoi(argv[2]) : 8;
  const int chunk_len = argc > 3 ? std::atoi(argv[3]) : 256;
  const float ratio = argc > 4 ? static_cast<float>(std::atof(argv[4])) : 0.15f;
  try {
    const frag_model_cfg cfg = frag::preset(preset);
    frag::Engine eng(cfg, 0, 1234);
    frag::ChunkStore store(cfg);
    frag::Rng rng(7);
    std::vector<frag::ChunkId> ids;
    for (int c = 0; c < n_chunks; ++c) {
      std::vector<frag::Token> chunk(chunk_len);
      for (auto& t : chunk) t = static_cast<frag::Token>(rng.below(cfg.vocab));
      ids.push_back(eng.preprocess_isolated(store, chunk));
    }
    std::vector<frag::Token> q(32);
    for (auto& t : q) t = static_cast<frag::Token>(rng.below(cfg.vocab));
    frag::Result res(eng, n_chunks * chunk_len + 32 + 16);  // + room for 16 decoded tokens
    frag_reprocess_opts opts{};
    opts.timing = 1;
    eng.reprocess(store, q, ids, ratio, res, {}, &opts);
    const auto t = res.timing();
    std::printf("preset=%s T=%d k=%zu first_token=%d ttft=%.3f ms (stitch %.3f, question %.3f, select %.3f, "
                "sparse %.3f, lm_head %.3f)\n",
                preset.c_str(), n_chunks * chunk_len + 32, res.critical_positions().size(), res.first_token(),
                t.total_ms, t.stitch_ms, t.question_ms, t.select_ms, t.sparse_ms, t.lm_head_ms);
    // sparse_prefill_and_decode: greedy answer over the fused cache
    const auto answer = eng.decode(res, 16);
    std::printf("answer:");
    for (auto tok : answer) std::printf(" %d", tok);
    std::printf("\n");
    const auto mem = res.memory();  // shared V pages: the chunks' V rows stay in the store's records
    std::printf("result memory %.1f MB, shared V pages %s\n", mem.first / 1e6, mem.second ? "yes" : "no");
    return 0;
  } catch (const frag::CudaError& e) {
    std::fprintf(stderr, "CudaError: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
