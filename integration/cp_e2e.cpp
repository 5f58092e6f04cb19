// End-to-end CP decomposition timing through the reference's own pipeline
// (pipeline.cpp::decompose, unchanged). Linked twice by integration/Makefile:
//   cp_e2e      -> against the B200 drop-in (facade over libxtsg.so)
//   cp_e2e_ref  -> against the reference library itself (oracle/_ref objects)
// so the two numbers differ only in the implementation of the hot path.
//
// usage: cp_e2e <I> <L> <R> <P> <S> <source: tensor|factors> [reps] [block]
// prints one JSON object per repetition with the four stage times
// (compression, decomposition, alignment, recovery), replica counts and the
// evaluate() errors against the generating factors.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "xts/pipeline.hpp"

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: %s I L R P S tensor|factors [reps] [block]\n", argv[0]);
    return 2;
  }
  const xts::index_t I = std::atoll(argv[1]), L = std::atoll(argv[2]), R = std::atoll(argv[3]);
  const xts::index_t P = std::atoll(argv[4]), S = std::atoll(argv[5]);
  const bool tensor = std::string(argv[6]) == "tensor";
  const int reps = argc > 7 ? std::atoi(argv[7]) : 1;
  const xts::index_t block = argc > 8 ? std::atoll(argv[8]) : 0;

  xts::SyntheticSpec spec;
  spec.dims = {I, I, I};
  spec.rank = R;
  spec.seed = 1;
  const xts::Synthetic syn = xts::generate(spec, tensor, std::uint64_t(1) << 36);
  for (int rep = 0; rep < reps; ++rep) {
    xts::PipelineConfig cfg;
    cfg.dims = {I, I, I};
    cfg.reduced = {L, L, L};
    cfg.rank = R;
    cfg.replicas = P;
    cfg.shared = S;
    cfg.block = {block, block, block};
    cfg.seed = 2;
    xts::RunMetrics m;
    const xts::TensorSource src =
        tensor ? xts::TensorSource::from_tensor(*syn.tensor) : xts::TensorSource::from_factors(syn.factors);
    const auto t0 = std::chrono::steady_clock::now();
    int status = 0;
    xts::FactorTriple rec;
    try {
      rec = xts::decompose(src, cfg, m);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "decompose failed: %s\n", e.what());
      status = 1;
    }
    const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double err[3] = {-1, -1, -1}, mse = -1;
    if (!status) {
      const xts::EvalReport ev = xts::evaluate(syn.factors, rec);
      for (int k = 0; k < 3; ++k) err[k] = ev.mode_rel_err[k];
      mse = ev.sample_mse;
    }
    std::printf(
        "{\"status\": %d, \"total_s\": %.6f, \"stages_s\": [%.6f, %.6f, %.6f, %.6f], \"replicas_total\": %lld, "
        "\"replicas_dropped\": %lld, \"factor_rel_err\": [%.3e, %.3e, %.3e], \"sample_mse\": %.3e}\n",
        status, total, m.stages[0].elapsed_s, m.stages[1].elapsed_s, m.stages[2].elapsed_s, m.stages[3].elapsed_s,
        static_cast<long long>(m.replicas_total), static_cast<long long>(m.replicas_dropped), err[0], err[1], err[2],
        mse);
    std::fflush(stdout);
  }
  return 0;
}
