// A C++ caller of the B200 library through the reference-shaped header only
// (include/dgnn/b200.hpp over include/dgnn_b200.h): synthesize a dynamic
// graph, train seq-first epochs or — with WORLD_SIZE > 1, one process per GPU
// — the window-sharded trainer with the NCCL gradient all-reduce, and print
// one JSON line per epoch (rank 0).
//
//   g++ -std=c++17 -I include examples/train_epoch.cpp -o train_epoch
//       -L paper_2501_15348_b200 -l:_dgnn_b200.so -Wl,-rpath,$PWD/paper_2501_15348_b200
//   (one command line)
//   ./train_epoch [nodes deg dim T edge_change feat_change arch hidden epochs]
//   WORLD_SIZE=2 RANK=r LOCAL_RANK=r DGNN_COMM_ID_FILE=/tmp/id ./train_epoch ...   (per rank)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "dgnn/b200.hpp"

namespace {

int env_int(const char* k, int dflt) {
  const char* v = std::getenv(k);
  return v ? std::atoi(v) : dflt;
}

// rank 0 writes the NCCL id to a file; the other ranks wait for it
std::vector<uint8_t> exchange_id(int rank, const std::string& path) {
  if (rank == 0) {
    std::vector<uint8_t> id = dgnn::Communicator::unique_id();
    const std::string tmp = path + ".tmp";
    std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<const char*>(id.data()), 128);
    std::rename(tmp.c_str(), path.c_str());
    return id;
  }
  std::vector<uint8_t> id(128);
  for (int i = 0; i < 6000; ++i) {
    std::ifstream f(path, std::ios::binary);
    if (f && f.read(reinterpret_cast<char*>(id.data()), 128)) return id;
    std::this_thread::sleep_for(std::chrono::milliseconds(10));
  }
  throw std::runtime_error("timed out waiting for the communicator id in " + path);
}

}  // namespace

int main(int argc, char** argv) {
  dgnn::SynthParams sp;
  sp.num_nodes = argc > 1 ? std::atoi(argv[1]) : 2000;
  sp.avg_degree = argc > 2 ? std::atof(argv[2]) : 8.0;
  sp.feature_dim = argc > 3 ? std::atoi(argv[3]) : 32;
  sp.num_snapshots = argc > 4 ? std::atoi(argv[4]) : 14;
  sp.edge_change_rate = argc > 5 ? std::atof(argv[5]) : 0.02;
  sp.feature_change_rate = argc > 6 ? std::atof(argv[6]) : 0.02;
  const int arch = argc > 7 ? std::atoi(argv[7]) : 3;
  const int hidden = argc > 8 ? std::atoi(argv[8]) : 64;
  const int epochs = argc > 9 ? std::atoi(argv[9]) : 2;
  const int world = env_int("WORLD_SIZE", 1), rank = env_int("RANK", 0);
  try {
    dgnn::detail::check_status(dgnn_set_device(env_int("LOCAL_RANK", 0)));
    dgnn::DynamicGraph graph = dgnn::synthesize(sp);
    dgnn::ModelConfig mcfg;
    mcfg.arch = static_cast<dgnn::Architecture>(arch);
    mcfg.hidden_dim = hidden;
    dgnn::TrainConfig tcfg;
    tcfg.epochs = epochs;
    std::vector<std::vector<double>> losses;
    std::vector<double> seconds;
    std::vector<double> params;
    if (world == 1 && env_int("DGNN_SEQ_FIRST", 0)) {
      dgnn::TrainSession s(graph, mcfg, tcfg);
      for (const dgnn::EpochReport& r : s.run()) {
        losses.push_back(r.sample_losses);
        seconds.push_back(r.seconds);
      }
      params = s.flatten_params();
    } else {
      std::unique_ptr<dgnn::Communicator> comm;
      if (world > 1) {
        const char* f = std::getenv("DGNN_COMM_ID_FILE");
        comm = std::make_unique<dgnn::Communicator>(exchange_id(rank, f ? f : "/tmp/dgnn_comm_id"), world,
                                                    rank);
      }
      dgnn::DistSession s(graph, mcfg, tcfg, world, rank, comm.get());
      for (int e = 0; e < epochs; ++e) {
        dgnn::EpochReport r = s.run_epoch();
        losses.push_back(r.sample_losses);
        seconds.push_back(r.seconds);
      }
      params = s.flatten_params();
    }
    // every rank prints its own line (its local window block's losses)
    std::printf("{\"rank\": %d, \"world\": %d, \"epochs\": [", rank, world);
    for (size_t e = 0; e < losses.size(); ++e) {
      std::printf("%s{\"seconds\": %.6f, \"sample_losses\": [", e ? ", " : "", seconds[e]);
      for (size_t i = 0; i < losses[e].size(); ++i) std::printf("%s%.17g", i ? ", " : "", losses[e][i]);
      std::printf("]}");
    }
    double psum = 0.0;
    for (double p : params) psum += p * p;
    std::printf("], \"num_params\": %zu, \"param_sq_sum\": %.17g, \"params_head\": [", params.size(), psum);
    for (size_t i = 0; i < params.size() && i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", params[i]);
    std::printf("]}\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "train_epoch: %s\n", e.what());
    return 1;
  }
  return 0;
}
