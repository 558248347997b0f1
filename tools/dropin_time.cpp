// Drop-in cost breakdown (profiling helper, not product code): compose / vp_set_scene (host slab
// upload) / output allocation / vp_render into pageable host memory, K=4096 M=16 at 1024^2.
// g++ -O2 -std=c++17 -Iinclude tools/dropin_time.cpp -Lpaper_2103_01954_b200 -lvpb -o /tmp/dropin_time
#include <chrono>
#include <cstdio>
#include <vector>
#include "vpb.h"
int main() {
  int k=4096,m=16,w=1024;
  std::vector<float> tr(size_t(k)*24), pay(size_t(k)*4*m*m*m), xf(size_t(k)*15);
  vp_make_shell_scene(k,m,tr.data(),pay.data());
  vp_ctx* c; vp_create(0,&c);
  auto T=[]{return std::chrono::duration<double,std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();};
  vp_camera cam; vp_shell_camera(-1,0,w,&cam);
  vp_march mc{}; mc.step_size=0.001f; mc.early_eps=0.01f;
  for (int it=0; it<4; ++it) {
    double t0=T(); vp_compose(k,tr.data(),xf.data()); double t1=T();
    vp_set_scene(c,k,m,xf.data(),pay.data(),8,8); double t2=T();
    std::vector<float> rgb(size_t(w)*w*3), a(size_t(w)*w); std::vector<int> s(size_t(w)*w); double t3=T();
    vp_render(c,&cam,&mc,rgb.data(),a.data(),s.data(),nullptr); double t4=T();
    printf("compose %.2f set_scene %.2f alloc %.2f render %.2f total %.2f\n", t1-t0,t2-t1,t3-t2,t4-t3,t4-t0);
  }
}
