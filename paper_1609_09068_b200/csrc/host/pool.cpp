// A persistent worker pool for the host builders' fork-join loops: the plan
// of a deep DAG runs thousands of short parallel phases (one per wavefront of
// the component DAG, one per BFS level), where spawning threads per phase
// costs more than the work.  One job at a time; a caller that finds the pool
// busy (another thread's plan, or a nested loop) runs on freshly spawned
// threads instead, so there is no deadlock and no shared state across jobs.
// Workers spin on the job counter for a short while after each job (phases
// follow each other within microseconds), then sleep on a condition variable.
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "parallel.hpp"

namespace levelrank {
inline namespace b200 {
namespace detail {
namespace {

class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 1; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  bool try_run(int t, void (*fn)(void*, int), void* arg) {
    std::unique_lock<std::mutex> busy(run_, std::try_to_lock);
    if (!busy.owns_lock()) return false;
    fn_ = fn;
    arg_ = arg;
    nt_ = t;
    pending_.store(static_cast<int>(workers_.size()));
    gen_.fetch_add(1);  // publishes the job (seq_cst)
    if (sleepers_.load() > 0) {
      std::lock_guard<std::mutex> lk(m_);
      cv_.notify_all();
    }
    fn(arg, 0);
    for (int spins = 0; pending_.load(std::memory_order_acquire) != 0; ++spins)
      if (spins > kSpin) std::this_thread::yield();
      else relax();
    return true;
  }

 private:
  // workers spin briefly between the many short phases of one plan, then sleep
  static constexpr int kSpin = 1 << 14;
  static void relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
  }
  void loop(int id) {
    unsigned long long seen = 0;
    for (;;) {
      unsigned long long g;
      int spins = 0;
      while ((g = gen_.load()) == seen && !stop_.load()) {
        if (++spins < kSpin) {
          relax();
          continue;
        }
        std::unique_lock<std::mutex> lk(m_);
        sleepers_.fetch_add(1);
        cv_.wait(lk, [&] { return gen_.load() != seen || stop_.load(); });
        sleepers_.fetch_sub(1);
        spins = 0;
      }
      if (stop_.load()) return;
      seen = g;
      if (id < nt_) fn_(arg_, id);
      pending_.fetch_sub(1, std::memory_order_release);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex run_, m_;
  std::condition_variable cv_;
  void (*fn_)(void*, int) = nullptr;
  void* arg_ = nullptr;
  int nt_ = 0;
  std::atomic<unsigned long long> gen_{0};
  std::atomic<int> pending_{0}, sleepers_{0};
  std::atomic<bool> stop_{false};
};

Pool& pool() {
  static Pool p(host_threads());
  return p;
}

}  // namespace

void pool_run_impl(int t, void (*fn)(void*, int), void* arg) {
  if (t <= 1) {
    fn(arg, 0);
    return;
  }
  Pool& p = pool();
  if (t <= p.size() && p.try_run(t, fn, arg)) return;
  std::vector<std::thread> ts;
  ts.reserve(static_cast<std::size_t>(t) - 1);
  for (int i = 1; i < t; ++i) ts.emplace_back([=] { fn(arg, i); });
  fn(arg, 0);
  for (auto& th : ts) th.join();
}

}  // namespace detail
}  // namespace b200
}  // namespace levelrank
