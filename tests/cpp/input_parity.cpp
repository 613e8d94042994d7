// C++ facade test of the input side (include/drb_rb.hpp: dataset, make_schedule,
// shard_batches, lockstep_batches), written the way the reference's trainer uses
// proj/src/scenario (trainer.cpp:93-113). Values come from the reference itself
// (tests/golden/input.json, tests/golden/drds_small.drds written by its write_dataset);
// gathered rows are compared with the file's own bytes. Exit code 0 = pass. Needs a GPU.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "../../include/drb_rb.hpp"

using namespace drb::b200;

#define EXPECT(cond)                                                                \
    do {                                                                            \
        if (!(cond)) {                                                              \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            return 1;                                                               \
        }                                                                           \
    } while (0)

int main(int argc, char** argv) {
    const std::string gold = argc > 1 ? argv[1] : "tests/golden";
    const std::string path = gold + "/drds_small.drds";

    // make_schedule(10, 4, 1) and shard_batches(arange(97)*3+1, 0, 4, 8, 1, 0, 0): input.json
    const auto sched = make_schedule(10, 4, 1);
    const std::vector<std::vector<std::uint32_t>> want_tasks = {{4, 2, 7}, {9, 0, 1}, {3, 6}, {5, 8}};
    EXPECT(sched.tasks == want_tasks);
    std::vector<std::size_t> td(97);
    for (std::size_t i = 0; i < td.size(); ++i)
        td[i] = i * 3 + 1;
    const auto batches = shard_batches(td, 0, 4, 8, 1, 0, 0);
    const std::vector<std::size_t> want_shard = {19, 37, 133, 22, 124, 214, 229, 67, 115, 205, 220, 187, 73,
                                                 235, 94, 43, 265, 286, 64, 289, 70, 79, 106, 199, 52};
    std::vector<std::size_t> flat;
    for (const auto& b : batches)
        flat.insert(flat.end(), b.begin(), b.end());
    EXPECT(batches.size() == 4 && flat == want_shard);
    EXPECT(lockstep_batches(97, 4, 8) == 3);  // smallest shard: 24 -> 3 (input.json)
    bool threw = false;
    try {
        shard_batches(td, 4, 4, 8, 1, 0, 0);
    } catch (const usage_error&) {
        threw = true;
    }
    EXPECT(threw);
    threw = false;
    try {
        make_schedule(10, 0, 1);
    } catch (const config_error&) {
        threw = true;
    }
    EXPECT(threw);

    // load_dataset + indices + device gather
    threw = false;
    try {
        dataset missing(gold + "/no_such.drds");
    } catch (const io_error& e) {
        threw = std::string(e.what()).find("cannot open dataset file") != std::string::npos;
    }
    EXPECT(threw);
    dataset ds(path);
    EXPECT(ds.size() == 40 && ds.feature_dim == 12 && ds.n_classes == 5 && ds.train_count == 35 &&
           ds.eval_count == 5);
    const auto train0 = ds.train_indices_of({0});
    EXPECT(train0.size() == 7 && train0[0] == 0 && train0[1] == 5);  // round-robin labels
    EXPECT(ds.eval_indices_of({0, 1}).size() == 2);

    std::ifstream f(path, std::ios::binary);
    const std::vector<unsigned char> file((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    const std::vector<std::uint64_t> idx = {0, 39, 5, 5, 17};
    const std::size_t S = ds.feature_dim * 4, rec = S + 4;
    std::uint64_t* d_idx;
    unsigned char* d_out;
    std::uint32_t* d_lab;
    EXPECT(cudaMalloc(&d_idx, idx.size() * 8) == cudaSuccess);
    EXPECT(cudaMalloc(&d_out, idx.size() * S) == cudaSuccess);
    EXPECT(cudaMalloc(&d_lab, idx.size() * 4) == cudaSuccess);
    EXPECT(cudaMemcpy(d_idx, idx.data(), idx.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess);
    const auto m = ds.gather(d_idx, std::uint32_t(idx.size()), d_out, d_lab);
    EXPECT(m.n == idx.size());
    std::vector<unsigned char> out(idx.size() * S);
    std::vector<std::uint32_t> lab(idx.size());
    EXPECT(cudaMemcpy(out.data(), d_out, out.size(), cudaMemcpyDeviceToHost) == cudaSuccess);
    EXPECT(cudaMemcpy(lab.data(), d_lab, lab.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess);
    for (std::size_t j = 0; j < idx.size(); ++j) {
        const unsigned char* r = file.data() + 22 + idx[j] * rec;
        EXPECT(std::memcmp(out.data() + j * S, r, S) == 0);
        std::uint32_t l;
        std::memcpy(&l, r + S, 4);
        EXPECT(lab[j] == l);
    }
    EXPECT(ds.device_error() == 0);
    // synth_dataset(5, 8, 12, 4.0, 11) is the fixture's content (written by the reference)
    const dataset syn = dataset::synth(5, 8, 12, 4.0, 11);
    EXPECT(syn.size() == ds.size() && syn.train_count == ds.train_count && syn.eval_count == ds.eval_count);
    void *fa, *fb;
    std::uint32_t *la, *lb;
    EXPECT(drb_ds_device_views(syn.raw(), &fa, &la) == DRB_OK && drb_ds_device_views(ds.raw(), &fb, &lb) == DRB_OK);
    std::vector<unsigned char> a(ds.size() * S), bb(ds.size() * S);
    EXPECT(cudaMemcpy(a.data(), fa, a.size(), cudaMemcpyDeviceToHost) == cudaSuccess);
    EXPECT(cudaMemcpy(bb.data(), fb, bb.size(), cudaMemcpyDeviceToHost) == cudaSuccess);
    EXPECT(a == bb);
    cudaFree(d_idx);
    cudaFree(d_out);
    cudaFree(d_lab);
    std::printf("input facade: schedule, shards, load, synth, indices, gather bit-exact\n");
    return 0;
}
