// A benchmark campaign written against the reference's bench.hpp API only: it compiles unchanged
// against the reference headers (oracle/Makefile builds that binary into oracle/_ref/campaign_ref)
// and against the drop-in (include/hpclust/bench.hpp over libhpcg.so -> examples/campaign_example);
// tests/test_campaign_gpu.py compares the two outputs series by series.
//   campaign_example <num_points> <features> <num_blobs> <max_samples> <n_exec> <algo,algo,...> <k,k,...>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>

#include <hpclust/bench.hpp>

static std::vector<std::string> split(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    for (std::string item; std::getline(ss, item, ',');)
        if (!item.empty()) out.push_back(item);
    return out;
}

static void put_summary(const char* name, const hpclust::MetricSummary& s) {
    std::printf("\"%s\": {\"median\": %.17g, \"min\": %.17g, \"max\": %.17g, \"stddev\": ", name, s.median, s.min, s.max);
    if (s.stddev)
        std::printf("%.17g}", *s.stddev);
    else
        std::printf("null}");
}

int main(int argc, char** argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: %s num_points features num_blobs max_samples n_exec algos ks\n", argv[0]);
        return 2;
    }
    try {
        hpclust::BlobSpec spec;
        spec.num_points = std::strtoull(argv[1], nullptr, 10);
        spec.features = std::strtoull(argv[2], nullptr, 10);
        spec.num_blobs = std::strtoull(argv[3], nullptr, 10);
        spec.center_min = -20.0;
        spec.center_max = 20.0;
        spec.std_min = 0.5;
        spec.std_max = 1.5;
        spec.noise_points = spec.num_points / 50;
        spec.noise_min = -25.0;
        spec.noise_max = 25.0;
        spec.seed = 5;
        const hpclust::BlobData data = hpclust::gen_blobs(spec);
        double checksum = 0.0;
        for (double v : data.points.values) checksum += v;

        if (std::string(argv[6]) == "metrics") {
            // host-only leg (no device): the metric helpers on values taken from the blob rows
            std::vector<hpclust::MetricRecord> recs;
            std::map<std::string, std::vector<double>> bests;
            std::vector<hpclust::WorkerState> workers(3);
            const auto& v = data.points.values;
            const int reps = std::atoi(argv[5]);
            for (int r = 0; r < reps; ++r) {
                hpclust::MetricRecord rec;
                rec.algorithm = "hybrid";
                rec.k = 7;
                rec.repetition = r;
                rec.epsilon = hpclust::relative_error(100.0 + v[(std::size_t)r], 100.0);
                rec.t = v[(std::size_t)(r + reps)];
                rec.n_d = (std::int64_t)(1000.0 * v[(std::size_t)(r + 2 * reps)]);
                if (r % 3) rec.t_bar = v[(std::size_t)(r + 3 * reps)];
                recs.push_back(rec);
                bests[r % 2 ? "a" : "b"].push_back(v[(std::size_t)(r + 4 * reps)]);
                workers[(std::size_t)r % 3].worker_id = r % 3;
                auto& tr = workers[(std::size_t)r % 3].update_trace;
                tr.push_back({(double)(r + 1), 50.0 - (double)tr.size() - 0.01 * r});
            }
            const hpclust::RunSeries s = hpclust::summarize(recs);
            const auto tb = hpclust::baseline_convergence_time(workers, 48.5);
            std::printf("{\"rows\": %zu, \"checksum\": %.17g, \"stds0\": %.17g, \"blob_last\": %d, ", data.points.rows,
                        checksum, data.stds[0], (int)data.blob_of_row[spec.num_points - 1]);
            put_summary("epsilon", s.epsilon);
            std::printf(", ");
            put_summary("t", s.t);
            std::printf(", ");
            put_summary("t_bar", *s.t_bar);
            std::printf(", \"n_d_median\": %.17g, \"f_bar\": %.17g, \"t_conv\": %.17g, \"default_s\": [%zu, %zu, %zu], "
                        "\"hybrid\": %d, \"known\": %zu}\n",
                        s.n_d_median, hpclust::baseline_objective(bests), tb ? *tb : -1.0,
                        hpclust::default_sample_size(1500), hpclust::default_sample_size(3000),
                        hpclust::default_sample_size(100000), (int)hpclust::is_hpclust_algorithm("hybrid"),
                        hpclust::all_algorithms().size());
            return 0;
        }
        hpclust::CampaignConfig cfg;
        cfg.dataset_name = "blobs";
        cfg.max_samples = std::strtoull(argv[4], nullptr, 10);
        cfg.n_exec = std::atoi(argv[5]);
        cfg.algorithms = split(argv[6]);
        for (const auto& k : split(argv[7])) cfg.k_list.push_back(std::strtoull(k.c_str(), nullptr, 10));
        cfg.master_seed = 2024;
        cfg.n_workers = 4;
        cfg.sample_size = 1500;
        cfg.segment_size = 2500;
        const std::vector<hpclust::RunSeries> series = hpclust::run_campaign(data.points, cfg);

        std::printf("{\"rows\": %zu, \"checksum\": %.17g, \"stds0\": %.17g, \"series\": [", data.points.rows, checksum,
                    data.stds[0]);
        for (std::size_t i = 0; i < series.size(); ++i) {
            const auto& s = series[i];
            std::printf("%s{\"dataset\": \"%s\", \"algorithm\": \"%s\", \"k\": %zu, ", i ? ", " : "", s.dataset.c_str(),
                        s.algorithm.c_str(), s.k);
            put_summary("epsilon", s.epsilon);
            std::printf(", ");
            put_summary("t", s.t);
            std::printf(", ");
            if (s.t_bar)
                put_summary("t_bar", *s.t_bar);
            else
                std::printf("\"t_bar\": null");
            std::printf(", \"n_d_median\": %.17g, \"n_s_median\": %.17g, \"sample_size\": %.17g, \"time_limit\": %.17g, "
                        "\"t1\": %.17g, \"t2\": %.17g, \"succ\": %s, \"records\": [",
                        s.n_d_median, s.n_s_median, s.sample_size, s.time_limit, s.t1, s.t2, s.succ ? "true" : "false");
            for (std::size_t r = 0; r < s.records.size(); ++r) {
                const auto& rec = s.records[r];
                std::printf("%s{\"rep\": %d, \"epsilon\": %.17g, \"t\": %.17g, \"n_d\": %lld, \"t_bar\": ", r ? ", " : "",
                            rec.repetition, rec.epsilon, rec.t, (long long)rec.n_d);
                if (rec.t_bar)
                    std::printf("%.17g}", *rec.t_bar);
                else
                    std::printf("null}");
            }
            std::printf("]}");
        }
        std::printf("]}\n");
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}
